# full GPU suite + bench lines (default, 1e-5, heavy t100) + ncu of k_pgd<0> (1e-5) and K2 count (default)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02q.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_r02q.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r02q.json 2> gpurun_out/bench_r02q.err; echo bench=$?
timeout 600 python bench.py --xi-rel 1e-5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_r02q_1e-5.json 2> gpurun_out/bench_r02q_1e-5.err; echo b5=$?
timeout 900 python bench.py --xi-rel 1.2e-4 --stop none --t-max 100 --steps 3 --warmup 3 --no-e2e --no-edit-log --no-cpu-baseline > gpurun_out/bench_r02q_t100.json 2> gpurun_out/bench_r02q_t100.err; echo bt=$?
for f in bench_r02q bench_r02q_1e-5 bench_r02q_t100; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f', d['value'], d['ms_per_step'], {k:round(x,2) for k,x in d['kernels_ms_per_step'].items()})"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pgd --launch-skip 200 --launch-count 1 -o gpurun_out/r02q_k3_1e-5 python bench.py --xi-rel 1e-5 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/ncu_k3.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pairs_count --launch-count 1 -o gpurun_out/r02q_k2 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/ncu_k2.log 2>&1; echo ncu2=$?
CC_K2_TILED=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pairs_count --launch-count 1 -o gpurun_out/r02q_k2_tiled python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/ncu_k2t.log 2>&1; echo ncu3=$?
