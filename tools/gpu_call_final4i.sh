# final bench lines of round 2 (default flags) at N = 1/2/4 on the final build
set -x
TAG=r02i
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/bench_${TAG}_n1.json 2> gpurun_out/bench_${TAG}_n1.err; echo n1=$?
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2968$N bench.py --gpus $N > gpurun_out/bench_${TAG}_n$N.json 2> gpurun_out/bench_${TAG}_n$N.err; echo n$N=$?
done
for N in 1 2 4; do python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_n$N.json'));print($N, d['value'], d['ms_per_step'], d.get('e2e',{}).get('value'), d['phases_ms'], d['roofline']['kernel'], d['roofline']['frac'], d['k3_roofline']['frac'], d['clocks'])"; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_${TAG}_ref.json 2> gpurun_out/bench_${TAG}_ref.err; echo ref=$?
