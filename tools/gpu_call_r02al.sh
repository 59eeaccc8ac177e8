# programmatic dependent launch for the PGD iteration kernels (default) vs plain launches (CC_PDL=0); 2 GPUs
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vranks.py tests/test_gpu_multi.py tests/test_gpu_edges.py -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_r02al.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_r02al.log
for v in 1 0 1 0; do
CC_PDL=$v CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02al_n1_$v.json 2> gpurun_out/bench_r02al_n1_$v.err
python -c "import json;d=json.load(open('gpurun_out/bench_r02al_n1_$v.json'));print('n1 pdl=$v', round(d['value'],1), round(d['ms_per_step'],2), d['phases_ms'])"
CC_PDL=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2964$v bench.py --gpus 2 --no-e2e --no-cpu-baseline --no-edit-log > gpurun_out/bench_r02al_n2_$v.json 2> gpurun_out/bench_r02al_n2_$v.err
python -c "import json;d=json.load(open('gpurun_out/bench_r02al_n2_$v.json'));print('n2 pdl=$v', round(d['value'],1), round(d['ms_per_step'],2), d['phases_ms'])"
done
