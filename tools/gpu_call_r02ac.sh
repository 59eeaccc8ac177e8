# K1 record stride A/B: 64-byte slots written in full (REC_STRIDE 2, default here) vs 32-byte records (rs1)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02ac.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu_r02ac.log
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02ac_$tag.json 2> gpurun_out/bench_r02ac_$tag.err; python -c "import json;d=json.load(open('gpurun_out/bench_r02ac_$tag.json'));k=d['kernels_ms_per_step'];print('$tag', round(d['value'],1), round(d['ms_per_step'],2), 'K1', k['K1_key'], k['K1_scatter'], k['K1_finish'])"; grep "memory in use" gpurun_out/bench_r02ac_$tag.err; }
for rep in 1 2; do
run rs2 CC_X=0
run rs1 CC_LIB_PATH=$PWD/variants/libcc_rs1.so
done
timeout 900 ncu --set full --clock-control none -k regex:"k_bin_scatter|k_row_finish" --launch-count 2 -o gpurun_out/r02ac_k1 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/ncu_k1rs.log 2>&1; echo ncu=$?
