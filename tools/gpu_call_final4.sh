# 4-GPU evidence: full GPU suite (incl. NCCL multi-rank), smoke, default bench at N = 1/2/4 and C5 at N = 2/4
set -x
TAG=${1:-r02f}
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu_${TAG}_4gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_${TAG}_4gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke=$?
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/bench_${TAG}_n1.json 2> gpurun_out/bench_${TAG}_n1.err; echo n1=$?
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N > gpurun_out/bench_${TAG}_n$N.json 2> gpurun_out/bench_${TAG}_n$N.err; echo n$N=$?
done
for N in 1 2 4; do python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_n$N.json'));print($N, d['value'], d['ms_per_step'], d.get('e2e',{}).get('value'), d.get('per_rank'), {k:round(x,1) for k,x in d['kernels_ms_per_step'].items()})"; done
for N in 4 2; do
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2956$N bench.py --gpus $N --config C5 --no-edit-log > gpurun_out/c5_${TAG}_n$N.json 2> gpurun_out/c5_${TAG}_n$N.err; echo c5n$N=$?
python -c "import json;d=json.load(open('gpurun_out/c5_${TAG}_n$N.json'));print('C5', $N, d['value'], d['ms_per_step'], d['result']['iterations'], d['result']['mcc_after'], d.get('per_rank'))"
done
