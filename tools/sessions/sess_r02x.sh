# session 4e: flattened traversal of the separable grid kernel; fp64 expansion kernel's cutoff on the high words
timeout 1500 python -m pytest tests/test_gpu_hotpath.py tests/test_gpu_mesh.py tests/test_gpu_fullsize.py tests/test_gpu_solver.py -x -q > gpurun_out/pytest_x.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_x.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('c4', d['ms_per_step'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['e2e']['ms_per_step'], d['detail']['rel_residual_true'], d['detail']['stage_ms_per_step'], d['detail']['isosurface']['ms'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"grid_sep_kernel" -c 1 -o gpurun_out/gridsep python tools/prof_grid.py c4 > gpurun_out/ncu_grid.log 2>&1; echo ncu_grid=$?
python tools/ncu_summary.py gpurun_out/gridsep.ncu-rep > gpurun_out/gridsep_ncu.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"sum_f64_syme" -c 1 -o gpurun_out/f64e python tools/prof_step.py c4 > gpurun_out/ncu_f64e.log 2>&1; echo ncu_f64e=$?
python tools/ncu_summary.py gpurun_out/f64e.ncu-rep > gpurun_out/f64e_ncu.txt 2>&1
