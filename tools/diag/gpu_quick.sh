set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/q_pytest.log
for v in solve sweep; do timeout 300 python tools/diag/post_time.py tools/diag/sweep/lib_$v.so C5 2>&1 | tail -1; done
