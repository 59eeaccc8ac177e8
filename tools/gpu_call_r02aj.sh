# K3 flattened chunk: NB = 2 entries per lane (variant nb2, smaller code) vs NB = 4 (default)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
run() { tag=$1; xi=$2; shift; shift; env "$@" timeout 600 python bench.py --xi-rel $xi --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02aj_$tag.json 2> gpurun_out/bench_r02aj_$tag.err; python -c "import json;d=json.load(open('gpurun_out/bench_r02aj_$tag.json'));k=d['kernels_ms_per_step'];print('$tag', round(d['value'],1), round(d['ms_per_step'],2), 'K3', k['K3_pgd'], d['result']['iterations'])"; }
for rep in 1 2; do
run nb4_5 1e-5 CC_X=0
run nb2_5 1e-5 CC_LIB_PATH=$PWD/variants/libcc_nb2.so
done
run nb4_6 1e-6 CC_X=0
run nb2_6 1e-6 CC_LIB_PATH=$PWD/variants/libcc_nb2.so
