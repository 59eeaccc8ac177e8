# warp-flattened fill pass + output writes only changed coordinates
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02ah.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_r02ah.log
for rep in 1 2; do
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02ah.json 2> gpurun_out/bench_r02ah.err
python -c "import json;d=json.load(open('gpurun_out/bench_r02ah.json'));print(round(d['value'],1), round(d['ms_per_step'],2), d['phases_ms'], {k:round(x,2) for k,x in d['kernels_ms_per_step'].items()})"
done
timeout 600 python bench.py --xi-rel 1e-5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02ah_1e-5.json 2> gpurun_out/bench_r02ah_1e-5.err
python -c "import json;d=json.load(open('gpurun_out/bench_r02ah_1e-5.json'));print('1e-5', round(d['value'],1), round(d['ms_per_step'],2), {k:round(x,2) for k,x in d['kernels_ms_per_step'].items()})"
