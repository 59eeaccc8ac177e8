# last round-2 check: full GPU suite on 4 GPUs (NCCL multi-rank incl.), smoke, bench N = 1/2/4, reference arm
set -x
TAG=r02j
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu_${TAG}_4gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu_${TAG}_4gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke=$?
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/bench_${TAG}_n1.json 2> gpurun_out/bench_${TAG}_n1.err; echo n1=$?
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2970$N bench.py --gpus $N > gpurun_out/bench_${TAG}_n$N.json 2> gpurun_out/bench_${TAG}_n$N.err; echo n$N=$?
done
for N in 1 2 4; do python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_n$N.json'));print($N, d['value'], d['ms_per_step'], d.get('e2e',{}).get('value'), d['phases_ms'], d['roofline']['frac'], d['k3_roofline']['frac'], d['clocks'])"; done
