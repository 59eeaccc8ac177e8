# output from the inputs + lazy slot_of + shared stable-forest cache in the warp count; full GPU suite; bench; ncu dense k_pgd<0> (1e-5)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02s.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_r02s.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r02s.json 2> gpurun_out/bench_r02s.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/bench_r02s.json'));print('default', d['value'], d['ms_per_step'], d['e2e'], {k:round(x,2) for k,x in d['kernels_ms_per_step'].items()})"
CC_K2_TILED=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02s_0.json 2> gpurun_out/bench_r02s_0.err; echo bench0=$?
python -c "import json;d=json.load(open('gpurun_out/bench_r02s_0.json'));print('perparticle', d['value'], d['ms_per_step'], d['kernels_ms_per_step']['K2_count'])"
grep "device memory" gpurun_out/bench_r02s.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pgd --launch-skip 20 --launch-count 1 -o gpurun_out/r02s_k3_dense python bench.py --xi-rel 1e-5 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/ncu_k3d.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pairs_count --launch-count 1 -o gpurun_out/r02s_k2w python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/ncu_k2w.log 2>&1; echo ncu2=$?
