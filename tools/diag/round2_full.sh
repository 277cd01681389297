#!/bin/bash
# Round-2 measurement pass on one B200: GPU tests, the bench line (with the CPU
# baseline), the reference arm, the ncu launch list of a short bench, and
# ncu --set full captures of K3 / K5 at C2 (exported to text).
python -m pytest tests -m gpu -q -ra > gpurun_out/r2_gputest.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.log 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_ref.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
  --log-file gpurun_out/r2_launches_raw.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-sampled \
  --no-scatter > gpurun_out/r2_ncu_launch.log 2>&1
bash tools/diag/ncu_captures.sh k3r2_c2:condense6_kernel:C2:none k5r2_c2:recover3:C2:none k4r2_c2:scatter_faces:C2:scatter
