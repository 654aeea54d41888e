python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_solver.py -q -x 2>&1 | tail -3
timeout 600 python tools/prof_precond.py c4 2>&1 | tail -1
timeout 600 python tools/prof_precond.py c4 200000 > gpurun_out/pp_plain.log 2>&1 && \
 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_precond.csv python tools/prof_precond.py c4 200000 > gpurun_out/ncu_pp.log 2>&1
tail -1 gpurun_out/pp_plain.log
