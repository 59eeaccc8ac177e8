# fused peer unpack + stop decision (k_peer_finish); 4 GPUs: multi-rank tests + bench N=1/2/4 + C5 N=4
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests/test_gpu_vranks.py tests/test_gpu_multi.py -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02ag.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_r02ag.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02ag_n1.json 2> gpurun_out/bench_r02ag_n1.err; echo n1=$?
for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N bench.py --gpus $N --no-edit-log > gpurun_out/bench_r02ag_n$N.json 2> gpurun_out/bench_r02ag_n$N.err; echo n$N=$?
done
for f in n1 n2 n4; do python -c "import json;d=json.load(open('gpurun_out/bench_r02ag_$f.json'));print('$f', round(d['value'],1), round(d['ms_per_step'],2), d['phases_ms'], d['per_rank'])"; done
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29619 bench.py --gpus 4 --config C5 --no-edit-log > gpurun_out/c5_r02ag_n4.json 2> gpurun_out/c5_r02ag_n4.err; echo c5n4=$?
python -c "import json;d=json.load(open('gpurun_out/c5_r02ag_n4.json'));print('C5', d['value'], d['ms_per_step'], d['result']['iterations'], d['result']['mcc_after'], d['phases_ms'], d.get('per_rank'))"
