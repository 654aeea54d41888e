# pool head-room reserved after the warm-up (rbf_pool_reserve): bench right after the pytest subset that reproduced the stretched steps, per-step trace with pool sizes
timeout 1500 python -m pytest tests/test_gpu_race_probe.py tests/test_gpu_loopback.py tests/test_gpu_solver.py tests/test_gpu_bench_slab.py -x -q > gpurun_out/pytest_d4.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_d4.log
for i in 1 2 3; do
RBF_BENCH_TRACE=1 timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench_$i.json')); print('run$i', d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['detail']['stage_ms_per_step'])"
grep "bench trace" gpurun_out/bench_$i.err | sed 's/\[bench trace\] step //' | tr '\n' ';' | cut -c1-900; echo
done
