# What the driver runs at round end, in its order: smoke(), the reference arm,
# the default bench, and both again under torchrun (one rank).
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/dl_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/dl_smoke.log
( time python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/dl_ref.json 2> gpurun_out/dl_ref.err ) 2>&1 | grep real; echo "ref rc=$?"
( time python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/dl_bench.json 2> gpurun_out/dl_bench.err ) 2>&1 | grep real; echo "bench rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/dl_tr.json 2> gpurun_out/dl_tr.err; echo "torchrun rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 5 --warmup 3 --split strong --config C5 --no-cpu-baseline > gpurun_out/dl_tr_c5.json 2> gpurun_out/dl_tr_c5.err; echo "torchrun c5 strong rc=$?"
head -c 300 gpurun_out/dl_ref.json; echo; head -c 300 gpurun_out/dl_bench.json; echo; head -c 300 gpurun_out/dl_tr.json; echo; head -c 300 gpurun_out/dl_tr_c5.json; echo
