set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v6_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/v6_pytest.log
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/v6_bench.json 2> gpurun_out/v6_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/v6_bench.json'));print(d['value'],d['kernels_ms'])"
