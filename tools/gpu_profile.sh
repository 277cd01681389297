# Round-end measurement: bench line (C2, default), ncu launch list of the same
# command, and one `ncu --set full` capture of each step kernel (C2).
set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"quad_build|condense6|recover3|geometry_kernel" -c 4 \
  -o gpurun_out/full_c2 python tools/diag/sweep_time.py paper_1305_1489_b200/libhdg_b200.so C2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
