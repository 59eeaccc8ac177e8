set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for V in cur noslot nokey; do
  if [ $V = cur ]; then unset CC_LIB_PATH; else export CC_LIB_PATH=$PWD/variants/libcc_$V.so; fi
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-edit-log --no-cpu-baseline > gpurun_out/ab_r02m_$V.json 2> gpurun_out/ab_r02m_$V.err; echo $V=$?
done
unset CC_LIB_PATH
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_run.py > gpurun_out/san_racecheck.log 2>&1; echo racecheck=$?
tail -5 gpurun_out/san_racecheck.log
