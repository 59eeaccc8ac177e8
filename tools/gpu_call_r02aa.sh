# K1 row finish on 32-bit x keys (64-bit only for rows with equal keys) vs the previous 64-bit network
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vranks.py tests/test_gpu_fullsize.py tests/test_gpu_edges.py -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02aa.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu_r02aa.log
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02aa_$tag.json 2> gpurun_out/bench_r02aa_$tag.err; python -c "import json;d=json.load(open('gpurun_out/bench_r02aa_$tag.json'));k=d['kernels_ms_per_step'];print('$tag', round(d['value'],1), round(d['ms_per_step'],2), 'K1', k['K1_key'], k['K1_scatter'], k['K1_finish'])"; }
for rep in 1 2; do
run k32 CC_X=0
run k64 CC_LIB_PATH=$PWD/variants/libcc_k64.so
done
