set -x
timeout 900 python -m pytest tests/test_gpu_invariants.py -m gpu -x -q > gpurun_out/q_inv.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/q_inv.log
python tools/diag/c6_clk.py tools/diag/sweep/lib_clk.so C2
python tools/diag/c6_clk.py tools/diag/sweep/lib_clk4.so C2
