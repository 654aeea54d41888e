# final build of round 2: full GPU suite, smoke, c4 bench (the driver's order), launch list, c5 and c3 lines
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
RBF_BENCH_TRACE=1 timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('c4', d['ms_per_step'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['e2e']['ms_per_step'], d['detail']['rel_residual_true'], d['detail']['stage_ms_per_step'], d['detail']['isosurface']['ms'])"
grep "bench trace" gpurun_out/bench.err | sed 's/\[bench trace\] step //' | cut -c1-8 | tr '\n' ' '; echo
timeout 300 python bench.py > gpurun_out/bench_default_flags.json 2> gpurun_out/bench_default_flags.err; echo bench_default_flags=$?
python -c "import json; d=json.load(open('gpurun_out/bench_default_flags.json')); print('default flags', d['steps'], d['warmup'], d['ms_per_step'], d['e2e']['ms_per_step'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e > gpurun_out/ncu.log 2>&1; echo ncu=$?
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench_c5=$?
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench_c3=$?
python -c "
import json
for c in ('c5','c3'):
    d=json.load(open('gpurun_out/bench_%s.json'%c)); print(c, d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['detail']['rel_residual_true'], d['detail']['stage_ms_per_step'])"
timeout 120 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo bench_ref=$?; head -c 400 gpurun_out/bench_ref.json
