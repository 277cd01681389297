set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v6_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/v6_pytest.log
bash tools/diag/time_variants.sh C4
HDG_K3_V3=1 python tools/diag/sweep_time.py tools/diag/sweep/lib_nw16.so C4 | sed 's/^/v3: /'
bash tools/diag/time_variants.sh C2 nw16
