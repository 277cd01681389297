#!/bin/bash
# One measurement pass on a B200 (gpurun -- 'bash tools/diag/measure_pass.sh PREFIX'):
# the GPU tests, a bench line per config, the ncu launch list of the default
# bench command (after it has run without ncu), and ncu --set full captures of
# the step kernels, exported to text under gpurun_out/ncu/. tools/diag/
# ncu_to_launches.py and ncu_details_summary.py turn the outputs into profiles/.
P=${1:-pass}
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -ra > gpurun_out/${P}_gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${P}_gputest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${P}_bench_c2.json 2> gpurun_out/${P}_bench_c2.err; echo "c2 rc=$?"
for c in C1 C3 C4 C5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/${P}_bench_$c.json 2> gpurun_out/${P}_bench_$c.err; echo "$c rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/${P}_launches_raw.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-sampled \
  --no-scatter > gpurun_out/${P}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
bash tools/diag/ncu_captures.sh k3v6_c2:condense6_kernel:C2:none k3v6_c4:condense6_kernel:C4:none k3v5_c3:condense5_kernel:C3:none \
  k7v3_c4:convection3_kernel:C4:conv k6_c5:postprocess2_kernel:C5:post k4_c2:scatter_faces:C2:scatter k5_c2:recover3:C2:none \
  k2_c2:quad_build:C2:none
