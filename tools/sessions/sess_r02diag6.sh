# reserve after the first warm-up step: bench after a pytest subset, trace; default flags
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_assembled.py -x -q > gpurun_out/pytest_d6.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_d6.log
for i in 1 2; do
RBF_BENCH_TRACE=1 timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench_$i.json')); print('run$i', d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['detail']['stage_ms_per_step'])"
grep "bench trace" gpurun_out/bench_$i.err | sed 's/\[bench trace\] step //' | tr '\n' ';' | cut -c1-900; echo
done
for i in 1 2; do
RBF_BENCH_TRACE=1 timeout 300 python bench.py > gpurun_out/bench_default_flags_$i.json 2> gpurun_out/bench_default_flags_$i.err; echo bench_default_flags=$?
python -c "import json; d=json.load(open('gpurun_out/bench_default_flags_$i.json')); print('default flags', d['steps'], d['warmup'], d['ms_per_step'], d['e2e']['ms_per_step'])"
grep "bench trace" gpurun_out/bench_default_flags_$i.err | sed 's/\[bench trace\] step //' | tr '\n' ';' | cut -c1-400; echo
done
