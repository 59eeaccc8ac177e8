# group-row 32-bit keys; full GPU suite; smoke; default bench (final single-GPU line)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02ab.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_r02ab.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02ab.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_r02ab.json 2> gpurun_out/bench_r02ab.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/bench_r02ab.json'));print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['k3_roofline']['frac'], d['cpu_baseline']['value'], d['clocks'], {k:round(x,2) for k,x in d['kernels_ms_per_step'].items()})"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_r02ab_ref.json 2> gpurun_out/bench_r02ab_ref.err; echo ref=$?
tail -c 300 gpurun_out/bench_r02ab_ref.json
