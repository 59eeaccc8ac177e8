set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu_r02g.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_r02g.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-edit-log --no-cpu-baseline > gpurun_out/bench_r02g.json 2> gpurun_out/bench_r02g.err; echo bench=$?
timeout 600 python bench.py --xi-rel 1e-6 --steps 3 --warmup 3 --no-e2e --no-edit-log --no-cpu-baseline > gpurun_out/bench_r02g_1e-6.json 2> gpurun_out/bench_r02g_1e-6.err; echo bench=$?
SCHED_REPS=1 CC_TMAX=30 timeout 600 python tools/sched_dump.py C4 1.2e-4 > gpurun_out/sched_c4_12e-4_r02g_t30.txt 2>&1 && \
SCHED_REPS=1 CC_TMAX=30 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pgd<.int.1>" -s 6 -c 1 -o gpurun_out/r02_k3_heavy_long python tools/sched_dump.py C4 1.2e-4 > gpurun_out/ncu_k3_heavy.log 2>&1; echo ncu=$?
