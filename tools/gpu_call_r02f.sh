set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -x --timeout 600 > gpurun_out/pytest_gpu_r02f.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_r02f.log
SCHED_REPS=1 CC_TMAX=1200 timeout 600 python tools/sched_dump.py C4 1.2e-4 > gpurun_out/sched_c4_12e-4_r02f.txt 2>&1; echo sched=$?
timeout 600 python bench.py --xi-rel 1e-6 --steps 1 --warmup 1 --no-e2e --no-edit-log --no-cpu-baseline > gpurun_out/bench_r02f_1e-6.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pairs|k_bin|k_cell|k_fof|k_union|k_flatten|k_mingid" -s 12 -c 14 -o gpurun_out/r02_k1k2k4_1e-6 python bench.py --xi-rel 1e-6 --steps 1 --warmup 1 --no-e2e --no-edit-log --no-cpu-baseline > gpurun_out/ncu_k1k2k4.log 2>&1; echo ncu=$?
