set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_codec.py -q -x --timeout 600 > gpurun_out/pytest_gpu_r02h.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_r02h.log
for V in cur lb0 lb6 oldv_lb0 oldv_lb4; do
  if [ $V = cur ]; then unset CC_LIB_PATH; else export CC_LIB_PATH=$PWD/variants/libcc_$V.so; fi
  timeout 600 python bench.py --xi-rel 1e-6 --steps 3 --warmup 3 --no-e2e --no-edit-log --no-cpu-baseline > gpurun_out/ab_r02h_$V.json 2> gpurun_out/ab_r02h_$V.err; echo $V=$?
done
