# K3 lean (one pair-term copy per site, out-of-line loss limbs and replay) vs full inlining, C4 1e-5 and 1e-6
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_vranks.py -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02t.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_r02t.log
for v in lean full lean full; do
if [ $v = full ]; then export CC_LIB_PATH=$PWD/variants/libcc_k3full.so; else unset CC_LIB_PATH; fi
timeout 600 python bench.py --xi-rel 1e-5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02t_$v.json 2> gpurun_out/bench_r02t_$v.err; echo b$v=$?
python -c "import json;d=json.load(open('gpurun_out/bench_r02t_$v.json'));print('$v 1e-5', d['value'], d['ms_per_step'], d['kernels_ms_per_step']['K3_pgd'], d['result']['iterations'])"
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02t6_$v.json 2> gpurun_out/bench_r02t6_$v.err
python -c "import json;d=json.load(open('gpurun_out/bench_r02t6_$v.json'));print('$v 1e-6', d['value'], d['ms_per_step'], d['kernels_ms_per_step']['K3_pgd'], d['result']['iterations'])"
done
unset CC_LIB_PATH
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pgd --launch-skip 20 --launch-count 1 -o gpurun_out/r02t_k3_dense python bench.py --xi-rel 1e-5 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/ncu_k3d.log 2>&1; echo ncu1=$?
