# stable forest moved out of the S2 count sweep (built at the first FoF labelling); full GPU suite + bench
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02v.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_r02v.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r02v.json 2> gpurun_out/bench_r02v.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/bench_r02v.json'));print('default', d['value'], d['ms_per_step'], d['incl_check'], d['e2e']['value'], {k:round(x,2) for k,x in d['kernels_ms_per_step'].items()}, d['pair_tests'], d['roofline'])"
timeout 600 python bench.py --xi-rel 1e-5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_r02v_1e-5.json 2> gpurun_out/bench_r02v_1e-5.err; echo b5=$?
python -c "import json;d=json.load(open('gpurun_out/bench_r02v_1e-5.json'));print('1e-5', d['value'], d['ms_per_step'], {k:round(x,2) for k,x in d['kernels_ms_per_step'].items()})"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pairs_count --launch-count 1 -o gpurun_out/r02v_k2deg python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/ncu_k2deg.log 2>&1; echo ncu=$?
