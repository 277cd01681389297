#!/bin/bash
# One-shot probe of the GPU box: FP64 peaks, host cores, Eigen availability.
set -x
mkdir -p gpurun_out
nproc > gpurun_out/probe_nproc.txt
lscpu > gpurun_out/probe_lscpu.txt
ls /usr/include/eigen3 > gpurun_out/probe_eigen.txt 2>&1
nvidia-smi > gpurun_out/probe_smi.txt 2>&1
./tools/microbench/fp64_peak > gpurun_out/probe_fp64.jsonl 2>&1
python - <<'PY' >> gpurun_out/probe_fp64.jsonl 2>&1
import torch, json
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
for _ in range(2): c = a @ b
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(5):
    s.record(); c = a @ b; e.record(); e.synchronize(); best = min(best, s.elapsed_time(e))
print(json.dumps({"probe": "cublas_dgemm_8192", "tflops": 2 * 8192**3 / best / 1e9}))
PY
