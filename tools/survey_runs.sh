# Bench lines for SURVEY §8(d)'s measurement workloads (N=1) + the default line, the reference
# arm and the launch list.  Usage under gpurun: bash tools/survey_runs.sh <tag>
TAG=${1:-r02}
OUT=gpurun_out/survey_$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
nvidia-smi -L > $OUT/gpu.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> $OUT/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > $OUT/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 $OUT/pytest_gpu.log
run() { name=$1; shift; timeout ${TO:-900} python bench.py "$@" > $OUT/$name.json 2> $OUT/$name.err; echo "$name rc=$?"; }
run default
run reference --impl reference
run C4_1e-5 --xi-rel 1e-5 --no-cpu-baseline --no-e2e
TO=1500 run C4_1.2e-4_capped --xi-rel 1.2e-4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-edit-log
run C4_1.2e-4_t100 --xi-rel 1.2e-4 --stop none --t-max 100 --steps 3 --warmup 3 --no-e2e --no-edit-log
run C1 --config C1 --no-e2e --no-edit-log
for xi in 1e-4 1e-3 1e-2; do run C2_$xi --config C2 --xi-rel $xi --t-max 2000 --no-e2e --no-edit-log; done
for xi in 1e-3 1e-4 1e-5 1e-6; do run C3_$xi --config C3 --xi-rel $xi --no-e2e --no-edit-log; done
python bench.py --steps 1 --warmup 1 --no-e2e --no-edit-log --no-cpu-baseline > $OUT/launch_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-edit-log --no-cpu-baseline > $OUT/ncu_launch.log 2>&1; echo ncu=$?
