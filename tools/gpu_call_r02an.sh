# K1 key pass with 4 particles (and 4 rank atomics in flight) per thread vs one (variant key1)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vranks.py tests/test_gpu_fullsize.py -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02an.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu_r02an.log
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02an_$tag.json 2> gpurun_out/bench_r02an_$tag.err; python -c "import json;d=json.load(open('gpurun_out/bench_r02an_$tag.json'));k=d['kernels_ms_per_step'];print('$tag', round(d['value'],1), round(d['ms_per_step'],2), 'K1', k['K1_key'], k['K1_scatter'], k['K1_finish'])"; }
for rep in 1 2; do
run key4 CC_X=0
run key1 CC_LIB_PATH=$PWD/variants/libcc_key1.so
done
