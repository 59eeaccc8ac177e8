# K2 count: warp-flattened (default) vs per-particle (CC_K2_TILED=0) + parity suites
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_vranks.py tests/test_gpu_fullsize.py tests/test_gpu_multi.py -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02r.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_r02r.log
for v in w 0 w 0; do
if [ $v = w ]; then unset CC_K2_TILED; else export CC_K2_TILED=0; fi
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02r_$v.json 2> gpurun_out/bench_r02r_$v.err; echo bench$v=$?
python -c "import json;d=json.load(open('gpurun_out/bench_r02r_$v.json'));print('$v', d['value'], d['ms_per_step'], d['kernels_ms_per_step']['K2_count'], d['pair_tests']['K2_count']['tests_per_step'], d['result']['n_pairs'], d['result']['fof_groups_orig'])"
done
unset CC_K2_TILED
timeout 900 python bench.py --xi-rel 1.2e-4 --stop none --t-max 100 --steps 2 --warmup 3 --no-e2e --no-edit-log --no-cpu-baseline > gpurun_out/bench_r02r_t100.json 2> gpurun_out/bench_r02r_t100.err; echo bt=$?
python -c "import json;d=json.load(open('gpurun_out/bench_r02r_t100.json'));print('t100', d['value'], d['ms_per_step'], {k:round(x,2) for k,x in d['kernels_ms_per_step'].items()})"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pairs_count --launch-count 1 -o gpurun_out/r02r_k2w python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/ncu_k2w.log 2>&1; echo ncu=$?
