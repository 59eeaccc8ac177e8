# K1 two-pass scatter, second form (8,192-particle tiles, 2^21-slot buckets)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
CC_K1_TWOPASS=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02z.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu_r02z.log
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02z_$tag.json 2> gpurun_out/bench_r02z_$tag.err; python -c "import json;d=json.load(open('gpurun_out/bench_r02z_$tag.json'));k=d['kernels_ms_per_step'];print('$tag', round(d['value'],1), round(d['ms_per_step'],2), 'K1', k['K1_key'], k['K1_scatter'], k['K1_finish'], 'K2', k['K2_count'])"; }
for rep in 1 2; do
run base CC_X=0
run twopass CC_K1_TWOPASS=1
done
CC_K1_TWOPASS=1 timeout 900 ncu --set full --clock-control none -k regex:"k_bin_bucket|k_bin_place" --launch-count 2 -o gpurun_out/r02z_k1tp python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/ncu_k1tp.log 2>&1; echo ncu=$?
