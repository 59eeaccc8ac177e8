# K2 count: proportional-guess window search (default) vs plain binary search (CC_K2_GUESS=0)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_vranks.py tests/test_gpu_fullsize.py -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02ai.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu_r02ai.log
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02ai_$tag.json 2> gpurun_out/bench_r02ai_$tag.err; python -c "import json;d=json.load(open('gpurun_out/bench_r02ai_$tag.json'));k=d['kernels_ms_per_step'];print('$tag', round(d['value'],1), round(d['ms_per_step'],2), 'K2_count', k['K2_count'], d['pair_tests']['K2_count']['tests_per_step'], d['result']['n_pairs'])"; }
for rep in 1 2; do
run guess CC_X=0
run binary CC_K2_GUESS=0
done
