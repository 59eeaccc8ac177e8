# C5 (1,073,734,015 particles, the paper's 256^3-box HACC hiRes shape, xi_rel = 1e-6) at R = 1, 2, 4
# and the default workload at R = 2, 4 (gpurun --gpus 4)
set -x
TAG=${1:-r02}
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for N in 4 2; do
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --config C5 --no-edit-log > gpurun_out/c5_${TAG}_n$N.json 2> gpurun_out/c5_${TAG}_n$N.err; echo c5n$N=$?
tail -c 400 gpurun_out/c5_${TAG}_n$N.json
done
CUDA_VISIBLE_DEVICES=0 timeout 1500 python bench.py --config C5 --no-edit-log > gpurun_out/c5_${TAG}_n1.json 2> gpurun_out/c5_${TAG}_n1.err; echo c5n1=$?
tail -c 400 gpurun_out/c5_${TAG}_n1.json; grep -i "memory\|error" gpurun_out/c5_${TAG}_n1.err | head -5
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N --no-edit-log > gpurun_out/bench_${TAG}_n$N.json 2> gpurun_out/bench_${TAG}_n$N.err; echo n$N=$?
done
