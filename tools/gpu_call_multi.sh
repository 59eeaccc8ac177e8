# Multi-GPU evidence (gpurun --gpus 4): the NCCL-rank parity tests (peer path and CC_PEER=0) and
# bench lines at R = 1, 2, 4 of the default workload.
set -x
TAG=${1:-r02}
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1800 python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py tests/test_gpu_edges.py -q --timeout 900 > gpurun_out/pytest_multi_$TAG.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_multi_$TAG.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-e2e --no-edit-log --no-cpu-baseline > gpurun_out/bench_${TAG}_n1.json 2> gpurun_out/bench_${TAG}_n1.err; echo n1=$?
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --no-edit-log > gpurun_out/bench_${TAG}_n$N.json 2> gpurun_out/bench_${TAG}_n$N.err; echo n$N=$?
done
