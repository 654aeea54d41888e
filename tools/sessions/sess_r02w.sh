# session 4d: pipelined persistent block-Jacobi apply
timeout 1500 python -m pytest tests/test_gpu_solver.py tests/test_gpu_loopback.py -x -q > gpurun_out/pytest_w.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_w.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('c4', d['ms_per_step'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['e2e']['ms_per_step'], d['detail']['rel_residual_true'], d['detail']['stage_ms_per_step'], d['detail']['isosurface']['ms'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"apply_sym" -s 3 -c 1 -o gpurun_out/apply python tools/prof_step.py c4 0 6 > gpurun_out/ncu_apply.log 2>&1; echo ncu_apply=$?
python tools/ncu_summary.py gpurun_out/apply.ncu-rep > gpurun_out/apply_ncu.txt 2>&1
