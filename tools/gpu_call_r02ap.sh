# K3 schedule at C4 1e-6 on the final build
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 python tools/sched_dump.py C4 1e-6 > gpurun_out/sched_c4_1e-6_r02ap.txt 2>&1; echo sched=$?
