# apply CTAs sized to the bin's largest block (64 .. 256 threads)
timeout 1500 python -m pytest tests/test_gpu_solver.py tests/test_gpu_loopback.py tests/test_gpu_race_probe.py -x -q > gpurun_out/pytest_aa.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_aa.log
for i in 1 2; do
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench_$i.json')); print('c4', d['ms_per_step'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['detail']['rel_residual_true'], d['detail']['stage_ms_per_step'])"
done
timeout 600 ncu --set full --clock-control none -k regex:"apply_sym" -s 12 -c 4 -o gpurun_out/apply python tools/prof_step.py c4 0 6 > gpurun_out/ncu_apply.log 2>&1; echo ncu_apply=$?
python tools/ncu_summary.py gpurun_out/apply.ncu-rep > gpurun_out/apply_ncu.txt 2>&1
