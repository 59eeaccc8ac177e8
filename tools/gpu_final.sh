set -x
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench1=$?
NG=$(nvidia-smi -L | wc -l)
if [ "$NG" -gt 1 ]; then
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $NG --no-e2e > gpurun_out/benchN.json 2> gpurun_out/benchN.err; echo benchN=$?
head -c 300 gpurun_out/benchN.json
fi
