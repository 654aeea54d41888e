# fp64 symmetric expansion form: parity (hotpath degenerate clouds, solver, fullsize c4 fp64 rows) + bench + ncu of it
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests/test_gpu_nlist.py tests/test_gpu_hotpath.py tests/test_gpu_solver.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_f64.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_f64.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('c4', d['ms_per_step'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['e2e']['ms_per_step'], d['detail']['rel_residual_true'], d['detail']['stage_ms_per_step'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sum_f64_syme -s 0 -c 1 -o gpurun_out/f64e python tools/prof_step.py c4 > gpurun_out/ncu_f64.log 2>&1; echo ncu=$?
ncu -i gpurun_out/f64e.ncu-rep --page raw --csv > gpurun_out/f64e_raw.csv 2>/dev/null; echo raw=$?
ncu -i gpurun_out/f64e.ncu-rep --page source --csv --print-source sass > gpurun_out/f64e_sass.csv 2>/dev/null; echo sass=$?
