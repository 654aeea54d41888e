# neighbour-list form of the symmetric fp32 operator: parity tests + c4 bench + ncu of the NL kernel
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests/test_gpu_nlist.py tests/test_gpu_hotpath.py -x -q > gpurun_out/pytest_nl.log 2>&1; echo pytest_nl=$?; tail -3 gpurun_out/pytest_nl.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('c4', d['ms_per_step'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['e2e']['ms_per_step'], d['detail']['rel_residual_true'], d['detail']['stage_ms_per_step'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sum_f32_symb -s 1 -c 1 -o gpurun_out/symb_nl python tools/prof_step.py c4 > gpurun_out/ncu_symb.log 2>&1; echo ncu=$?
ncu -i gpurun_out/symb_nl.ncu-rep --page source --csv --print-source sass > gpurun_out/symb_nl_sass.csv 2>/dev/null; echo sass=$?
ncu -i gpurun_out/symb_nl.ncu-rep --page raw --csv > gpurun_out/symb_nl_raw.csv 2>/dev/null; echo raw=$?
timeout 1500 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_ipc.py tests/test_gpu_fullsize.py tests/test_gpu_solver.py -x -q > gpurun_out/pytest_rest.log 2>&1; echo pytest_rest=$?; tail -3 gpurun_out/pytest_rest.log
