set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for K in 2 0.5 0.1 0.03; do
timeout 600 python bench.py --xi-rel 1e-6 --cells-per-particle $K --steps 3 --warmup 3 --no-e2e --no-edit-log --no-cpu-baseline > gpurun_out/bench_r02e_1e-6_K$K.json 2> gpurun_out/bench_r02e_1e-6_K$K.err; echo bench=$?
done
timeout 600 python bench.py --xi-rel 1e-5 --cells-per-particle 0.1 --steps 3 --warmup 3 --no-e2e --no-edit-log --no-cpu-baseline > gpurun_out/bench_r02e_1e-5_K0.1.json 2> gpurun_out/bench_r02e_1e-5_K0.1.err; echo bench=$?
timeout 600 python bench.py --steps 1 --warmup 1 --no-e2e --no-edit-log --no-cpu-baseline > gpurun_out/bench_r02e_plain.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pgd -s 6 -c 2 -o gpurun_out/r02_k3_dense python bench.py --steps 1 --warmup 1 --no-e2e --no-edit-log --no-cpu-baseline > gpurun_out/ncu_k3_dense.log 2>&1; echo ncu=$?
