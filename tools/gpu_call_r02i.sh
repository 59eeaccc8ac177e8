set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for V in cur slotorder xorder; do
  if [ $V = cur ]; then unset CC_LIB_PATH; else export CC_LIB_PATH=$PWD/variants/libcc_$V.so; fi
  SCHED_REPS=1 CC_TMAX=40 timeout 600 python tools/sched_dump.py C4 1.2e-4 > gpurun_out/ab_r02i_sched_$V.txt 2>&1; echo sched_$V=$?
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-edit-log --no-cpu-baseline > gpurun_out/ab_r02i_$V.json 2> gpurun_out/ab_r02i_$V.err; echo $V=$?
done
unset CC_LIB_PATH
SCHED_REPS=1 CC_TMAX=12 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pgd -s 7 -c 1 -o gpurun_out/r02_k3_heavy_long python tools/sched_dump.py C4 1.2e-4 > gpurun_out/ncu_k3_heavy.log 2>&1; echo ncu=$?
