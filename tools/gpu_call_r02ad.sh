# multi-GPU phase attribution: N=1 and N=2 (peer path and CC_PEER=0)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02ad_n1.json 2> gpurun_out/bench_r02ad_n1.err; echo n1=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 2 --no-e2e --no-edit-log > gpurun_out/bench_r02ad_n2.json 2> gpurun_out/bench_r02ad_n2.err; echo n2=$?
CC_PEER=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29572 bench.py --gpus 2 --no-e2e --no-edit-log > gpurun_out/bench_r02ad_n2np.json 2> gpurun_out/bench_r02ad_n2np.err; echo n2np=$?
for f in n1 n2 n2np; do python -c "import json;d=json.load(open('gpurun_out/bench_r02ad_$f.json'));print('$f', round(d['value'],1), round(d['ms_per_step'],2), d['phases_ms'], d['per_rank'])"; done
