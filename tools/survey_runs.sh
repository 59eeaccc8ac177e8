# Bench lines for SURVEY §8(d)'s measurement workloads (N=1): C1, C2 xi sweep, C3 xi sweep,
# C4 at xi_rel 1.2e-4 (density-matched heavy case) and 1e-6.  Usage under gpurun:
#   bash tools/survey_runs.sh <tag>
TAG=${1:-r02}
OUT=gpurun_out/survey_$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
nvidia-smi -L > $OUT/gpu.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> $OUT/gpu.txt
run() { name=$1; shift; timeout ${TO:-900} python bench.py --steps 3 --warmup 3 --no-e2e --no-edit-log "$@" > $OUT/$name.json 2> $OUT/$name.err; echo "$name rc=$?"; }
run C1 --config C1 --no-cpu-baseline
for xi in 1e-4 1e-3 1e-2; do run C2_$xi --config C2 --xi-rel $xi --no-cpu-baseline --t-max 2000; done
for xi in 1e-3 1e-4 1e-5 1e-6; do run C3_$xi --config C3 --xi-rel $xi --no-cpu-baseline; done
run C4_1e-6 --config C4 --xi-rel 1e-6 --no-cpu-baseline
TO=1500 run C4_1.2e-4 --config C4 --xi-rel 1.2e-4 --no-cpu-baseline
