# A/B of the staged (shared-memory) K2 count against the per-particle form + K2 parity tests
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_vranks.py tests/test_gpu_fullsize.py tests/test_gpu_multi.py -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02p.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_r02p.log
for v in 1 0 1 0; do
CC_K2_TILED=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02p_t$v.json 2> gpurun_out/bench_r02p_t$v.err; echo bench$v=$?
python -c "import json;d=json.load(open('gpurun_out/bench_r02p_t$v.json'));print('tiled=$v', d['value'], d['ms_per_step'], {k:round(x,2) for k,x in d['kernels_ms_per_step'].items() if k.startswith('K2')}, d['pair_tests'])"
done
CC_K2_TILED=1 timeout 600 python bench.py --xi-rel 1e-5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02p_1e-5.json 2>&1; echo b5=$?
python -c "import json;d=json.load(open('gpurun_out/bench_r02p_1e-5.json'));print('1e-5', d['value'], d['ms_per_step'], {k:round(x,2) for k,x in d['kernels_ms_per_step'].items() if k.startswith('K2')})"
