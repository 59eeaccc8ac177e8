set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02o.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu_r02o.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r02o.json 2> gpurun_out/bench_r02o.err; echo bench=$?
timeout 600 python bench.py --xi-rel 1e-5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_r02o_1e-5.json 2> gpurun_out/bench_r02o_1e-5.err; echo bench=$?
