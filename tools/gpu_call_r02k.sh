set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02k.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu_r02k.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-edit-log --no-cpu-baseline > gpurun_out/bench_r02k.json 2> gpurun_out/bench_r02k.err; echo bench=$?
timeout 600 python bench.py --xi-rel 1e-5 --steps 3 --warmup 3 --no-e2e --no-edit-log --no-cpu-baseline > gpurun_out/bench_r02k_1e-5.json 2> gpurun_out/bench_r02k_1e-5.err; echo bench=$?
for K in 0.03 0.1; do timeout 600 python bench.py --cells-per-particle $K --steps 3 --warmup 3 --no-e2e --no-edit-log --no-cpu-baseline > gpurun_out/bench_r02k_K$K.json 2> gpurun_out/bench_r02k_K$K.err; echo benchK=$?; done
SCHED_REPS=1 CC_TMAX=1200 timeout 600 python tools/sched_dump.py C4 1.2e-4 > gpurun_out/sched_c4_12e-4_r02k.txt 2>&1; echo sched=$?
