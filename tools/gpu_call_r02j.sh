set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu_r02j.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_r02j.log
SCHED_REPS=1 CC_TMAX=1200 timeout 600 python tools/sched_dump.py C4 1.2e-4 > gpurun_out/sched_c4_12e-4_r02j.txt 2>&1; echo sched=$?
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-edit-log --no-cpu-baseline > gpurun_out/bench_r02j.json 2> gpurun_out/bench_r02j.err; echo bench=$?
