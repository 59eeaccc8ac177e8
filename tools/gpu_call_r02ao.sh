# warning cleanup check: full 1-GPU suite, smoke, default bench
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02ao.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu_r02ao.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02ao.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_r02ao.json 2> gpurun_out/bench_r02ao.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/bench_r02ao.json'));print(d['value'], d['ms_per_step'], d['e2e']['value'], d['gpu_launches'], d['clocks'])"
