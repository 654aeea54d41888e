# session 4c: grid staging on the kernel's own rings, dot kernel at 3 CTAs/SM, apply rows on 4 accumulators
timeout 1500 python -m pytest tests/test_gpu_hotpath.py tests/test_gpu_solver.py tests/test_gpu_mesh.py tests/test_gpu_loopback.py -x -q > gpurun_out/pytest_v.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_v.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('c4', d['ms_per_step'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['e2e']['ms_per_step'], d['detail']['rel_residual_true'], d['detail']['stage_ms_per_step'], d['detail']['isosurface']['ms'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"grid_sep_kernel" -c 1 -o gpurun_out/gridsep python tools/prof_grid.py c4 > gpurun_out/ncu_grid.log 2>&1; echo ncu_grid=$?
python tools/ncu_summary.py gpurun_out/gridsep.ncu-rep > gpurun_out/gridsep_ncu.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"apply_sym_kernel" -s 3 -c 1 -o gpurun_out/apply python tools/prof_step.py c4 0 6 > gpurun_out/ncu_apply.log 2>&1; echo ncu_apply=$?
python tools/ncu_summary.py gpurun_out/apply.ncu-rep > gpurun_out/apply_ncu.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"multi_dot4" -s 38 -c 2 -o gpurun_out/dot python tools/prof_step.py c4 0 42 > gpurun_out/ncu_dot.log 2>&1; echo ncu_dot=$?
python tools/ncu_summary.py gpurun_out/dot.ncu-rep > gpurun_out/dot_ncu.txt 2>&1
