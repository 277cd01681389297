#!/bin/bash
# Round-2 (final session) measurement pass: GPU tests, bench lines for every
# config, the ncu launch list of the default bench, ncu --set full of K3 v6.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -ra > gpurun_out/r2d_gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2d_gputest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2d_bench_c2.json 2> gpurun_out/r2d_bench_c2.err; echo "c2 rc=$?"
for c in C1 C3 C4 C5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r2d_bench_$c.json 2> gpurun_out/r2d_bench_$c.err; echo "$c rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/r2d_launches_raw.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-sampled \
  --no-scatter > gpurun_out/r2d_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
bash tools/diag/ncu_captures.sh k3v6_c2:condense6_kernel:C2:none k3v6_c4:condense6_kernel:C4:none k6_c5:postprocess2_kernel:C5:post
