# initial / final PGD statistics from the trace (no separate counting passes on a converged run); 2 GPUs
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 2000 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02am.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_r02am.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02am.log 2>&1; echo smoke=$?
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02am_n1.json 2> gpurun_out/bench_r02am_n1.err; echo n1=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 2 --no-edit-log > gpurun_out/bench_r02am_n2.json 2> gpurun_out/bench_r02am_n2.err; echo n2=$?
for f in n1 n2; do python -c "import json;d=json.load(open('gpurun_out/bench_r02am_$f.json'));print('$f', round(d['value'],1), round(d['ms_per_step'],2), d['phases_ms'], d['result'])"; done
