# multi-GPU K3 iteration periods (2 and 4 ranks, C4 default)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2963$N tools/sched_multi.py C4 > gpurun_out/sched_multi_n$N.txt 2>&1; echo n$N=$?
grep -E "iterations|kernel stats" gpurun_out/sched_multi_n$N.txt | head -8
done
