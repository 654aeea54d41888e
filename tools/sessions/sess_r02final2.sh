# final round-2 check, part 2: SPD Gauss-Jordan assembly with fp32-tier entries (solver / quality / full-size tests, c4 bench, launch list)
timeout 1800 python -m pytest tests/test_gpu_solver.py tests/test_gpu_quality.py tests/test_gpu_fullsize.py tests/test_gpu_loopback.py tests/test_gpu_race_probe.py -x -q > gpurun_out/pytest_f2.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_f2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('c4', d['ms_per_step'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['e2e']['ms_per_step'], d['detail']['rel_residual_true'], d['detail']['stage_ms_per_step'], d['detail']['isosurface']['ms'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e > gpurun_out/ncu.log 2>&1; echo ncu=$?
timeout 600 ncu --set full --clock-control none -k regex:"gj_spd" -c 4 -o gpurun_out/gj python tools/prof_step.py c4 0 3 > gpurun_out/ncu_gj.log 2>&1; echo ncu_gj=$?
python tools/ncu_summary.py gpurun_out/gj.ncu-rep > gpurun_out/gj_ncu.txt 2>&1
