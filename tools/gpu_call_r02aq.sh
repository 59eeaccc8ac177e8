# k_tail entry / capacity / block-count A/B (variants tailmid: enter 16K cap 64K; tailbig: enter 32K cap 128K, 148 blocks)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
CC_LIB_PATH=$PWD/variants/libcc_tailbig.so timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02aq.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu_r02aq.log
run() { tag=$1; xi=$2; shift; shift; env "$@" timeout 600 python bench.py --xi-rel $xi --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02aq_$tag.json 2> gpurun_out/bench_r02aq_$tag.err; python -c "import json;d=json.load(open('gpurun_out/bench_r02aq_$tag.json'));k=d['kernels_ms_per_step'];print('$tag', round(d['value'],1), round(d['ms_per_step'],2), 'K3', k['K3_pgd'])"; }
for rep in 1 2; do
run base6 1e-6 CC_X=0
run mid6 1e-6 CC_LIB_PATH=$PWD/variants/libcc_tailmid.so
run big6 1e-6 CC_LIB_PATH=$PWD/variants/libcc_tailbig.so
done
run base5 1e-5 CC_X=0
run mid5 1e-5 CC_LIB_PATH=$PWD/variants/libcc_tailmid.so
run big5 1e-5 CC_LIB_PATH=$PWD/variants/libcc_tailbig.so
