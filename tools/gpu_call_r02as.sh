# PGD iteration 1 builds the frontier bitmaps (iteration 2 selects) vs round-1 behaviour (variant bld0)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_vranks.py tests/test_gpu_fullsize.py -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02as.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu_r02as.log
run() { tag=$1; xi=$2; shift; shift; env "$@" timeout 600 python bench.py --xi-rel $xi --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02as_$tag.json 2> gpurun_out/bench_r02as_$tag.err; python -c "import json;d=json.load(open('gpurun_out/bench_r02as_$tag.json'));k=d['kernels_ms_per_step'];print('$tag', round(d['value'],1), round(d['ms_per_step'],2), 'K3', k['K3_pgd'], d['result']['iterations'])"; }
for rep in 1 2; do
run bld1_6 1e-6 CC_X=0
run bld0_6 1e-6 CC_LIB_PATH=$PWD/variants/libcc_bld0.so
done
run bld1_5 1e-5 CC_X=0
run bld0_5 1e-5 CC_LIB_PATH=$PWD/variants/libcc_bld0.so
