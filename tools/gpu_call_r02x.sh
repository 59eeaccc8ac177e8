# clamp-still freeze (frontier) : full GPU suite + bench default / 1e-5 / t100 heavy + schedule
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02x.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_r02x.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r02x.json 2> gpurun_out/bench_r02x.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/bench_r02x.json'));print('default', d['value'], d['ms_per_step'], d['result']['iterations'], {k:round(x,2) for k,x in d['kernels_ms_per_step'].items()}, d['roofline'])"
timeout 600 python bench.py --xi-rel 1e-5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_r02x_1e-5.json 2> gpurun_out/bench_r02x_1e-5.err; echo b5=$?
python -c "import json;d=json.load(open('gpurun_out/bench_r02x_1e-5.json'));print('1e-5', d['value'], d['ms_per_step'], d['result']['iterations'], {k:round(x,2) for k,x in d['kernels_ms_per_step'].items()})"
timeout 900 python bench.py --xi-rel 1.2e-4 --stop none --t-max 100 --steps 2 --warmup 3 --no-e2e --no-edit-log --no-cpu-baseline > gpurun_out/bench_r02x_t100.json 2> gpurun_out/bench_r02x_t100.err; echo bt=$?
python -c "import json;d=json.load(open('gpurun_out/bench_r02x_t100.json'));print('t100', d['value'], d['ms_per_step'], {k:round(x,2) for k,x in d['kernels_ms_per_step'].items()})"
timeout 600 python tools/sched_dump.py C4 1e-6 > gpurun_out/sched_c4_1e-6_r02x.txt 2>&1; echo sched=$?
timeout 900 python tools/sched_dump.py C4 1e-5 > gpurun_out/sched_c4_1e-5_r02x.txt 2>&1; echo sched5=$?
