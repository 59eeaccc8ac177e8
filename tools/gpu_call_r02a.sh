set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r02a.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu_r02a.log
export SCHED_REPS=1 CC_TMAX=1200
timeout 600 python tools/sched_dump.py C4 1.2e-4 > gpurun_out/sched_c4_12e-4_t1200.txt 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_pgd -s 1000 -c 2 -o gpurun_out/r02_k3_tail python tools/sched_dump.py C4 1.2e-4 > gpurun_out/ncu_k3_tail.log 2>&1; echo ncu=$?
