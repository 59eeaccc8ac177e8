# k_tail from 32K-editable lists on 148 blocks (adopted) + a 128K/512K variant; full suite, multi-rank, bench
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu_r02ar.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu_r02ar.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02ar.log 2>&1; echo smoke=$?
run() { tag=$1; xi=$2; shift; shift; env "$@" timeout 600 python bench.py --xi-rel $xi --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02ar_$tag.json 2> gpurun_out/bench_r02ar_$tag.err; python -c "import json;d=json.load(open('gpurun_out/bench_r02ar_$tag.json'));k=d['kernels_ms_per_step'];print('$tag', round(d['value'],1), round(d['ms_per_step'],2), 'K3', k['K3_pgd'])"; }
for rep in 1 2; do
run big6 1e-6 CC_X=0
run huge6 1e-6 CC_LIB_PATH=$PWD/variants/libcc_tailhuge.so
done
run big5 1e-5 CC_X=0
run huge5 1e-5 CC_LIB_PATH=$PWD/variants/libcc_tailhuge.so
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2967$N bench.py --gpus $N --no-edit-log > gpurun_out/bench_r02ar_n$N.json 2> gpurun_out/bench_r02ar_n$N.err; echo n$N=$?
python -c "import json;d=json.load(open('gpurun_out/bench_r02ar_n$N.json'));print($N, d['value'], d['ms_per_step'])"
done
