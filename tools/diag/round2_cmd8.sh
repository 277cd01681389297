for v in base t2w1e8 t2w1e16 t2w2e8; do python tools/diag/sweep_time.py tools/diag/sweep/lib_$v.so C4; done > gpurun_out/variants.log 2>&1
for v in base t3w1e8; do python tools/diag/sweep_time.py tools/diag/sweep/lib_$v.so C2; done >> gpurun_out/variants.log 2>&1
bash tools/diag/ncu_captures.sh
