# K3 traffic capture (iteration 1 at the default workload), K3 schedule at 1e-6, K1 kernels ncu
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 python tools/sched_dump.py C4 1e-6 > gpurun_out/sched_c4_1e-6_r02w.txt 2>&1; echo sched=$?
tail -5 gpurun_out/sched_c4_1e-6_r02w.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pgd --launch-skip 2 --launch-count 2 -o gpurun_out/r02w_k3_it1 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/ncu_k3it1.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bin_scatter|k_row_finish|k_bin_key" --launch-count 3 -o gpurun_out/r02w_k1 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/ncu_k1.log 2>&1; echo ncu2=$?
