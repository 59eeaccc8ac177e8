set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 python -m pytest tests/test_gpu_codec.py -x -q > gpurun_out/pytest_codec.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_codec.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
tail -3 gpurun_out/smoke.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 2 > gpurun_out/bench_codec.json 2> gpurun_out/bench_codec.err; echo bench=$?
tail -5 gpurun_out/bench_codec.err
