# final round-2 check on one B200: GPU suite, smoke, c4 bench, launch list, ncu --set full of the dominant kernel and of the apply bins, c5 and c3 lines
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('c4', d['ms_per_step'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['e2e']['ms_per_step'], d['detail']['rel_residual_true'], d['detail']['stage_ms_per_step'], d['detail']['isosurface']['ms'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e > gpurun_out/ncu.log 2>&1; echo ncu=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sum_f32_symb -s 2 -c 1 -o gpurun_out/symb_full python tools/prof_step.py c4 0 6 > gpurun_out/ncu_symb.log 2>&1; echo ncu_symb=$?
python tools/ncu_summary.py gpurun_out/symb_full.ncu-rep > gpurun_out/symb_ncu.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"apply_sym" -s 12 -c 4 -o gpurun_out/apply python tools/prof_step.py c4 0 6 > gpurun_out/ncu_apply.log 2>&1; echo ncu_apply=$?
python tools/ncu_summary.py gpurun_out/apply.ncu-rep > gpurun_out/apply_ncu.txt 2>&1
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench_c5=$?
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench_c3=$?
python -c "
import json
for c in ('c5','c3'):
    d=json.load(open('gpurun_out/bench_%s.json'%c)); print(c, d['ms_per_step'], d['roofline']['frac'], d['detail']['rel_residual_true'], d['detail']['stage_ms_per_step'])"
