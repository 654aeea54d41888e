# reproduce the stretched cells stage (bench right after a pytest subset) and look at the box: load average, memory, GPU processes, per-step trace
timeout 1500 python -m pytest tests/test_gpu_race_probe.py tests/test_gpu_loopback.py -x -q > gpurun_out/pytest_d2.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_d2.log
uptime; free -m | head -2; nvidia-smi --query-compute-apps=pid,used_memory --format=csv,noheader; ps -eo pid,pcpu,etime,cmd --sort=-pcpu | head -5
RBF_BENCH_TRACE=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench_a.json')); print('after-pytest', d['ms_per_step'], d['clocks'].get('samples'), d['detail']['stage_ms_per_step'])"
grep "bench trace" gpurun_out/bench_a.err | tr '\n' ';' | cut -c1-700; echo
uptime
RBF_BENCH_NO_CLOCKS=1 RBF_BENCH_TRACE=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench_b.json')); print('noclocks', d['ms_per_step'], d['detail']['stage_ms_per_step'])"
grep "bench trace" gpurun_out/bench_b.err | tr '\n' ';' | cut -c1-700; echo
