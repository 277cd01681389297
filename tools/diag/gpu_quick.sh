set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/q_pytest.log
bash tools/diag/time_variants.sh C3
