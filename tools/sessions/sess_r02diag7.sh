# after pre-creating the profiling events (rbf_profile_enable): the reproduction of the step-8..10 stall (heavy pytest subset first), without and with the sampler
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_assembled.py -x -q > gpurun_out/pytest_d7.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_d7.log
for mode in noclocks default default2 default3; do
  case $mode in
    noclocks*) export RBF_BENCH_NO_CLOCKS=1;;
    lms1000) unset RBF_BENCH_NO_CLOCKS; export RBF_BENCH_CLOCKS_MS=1000;;
    *) unset RBF_BENCH_NO_CLOCKS; unset RBF_BENCH_CLOCKS_MS;;
  esac
  RBF_BENCH_TRACE=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_$mode.json 2> gpurun_out/bench_$mode.err; echo bench=$?
  python -c "import json; d=json.load(open('gpurun_out/bench_$mode.json')); print('$mode', d['ms_per_step'], d['detail']['stage_ms_per_step']['cells'])"
  grep "bench trace" gpurun_out/bench_$mode.err | sed 's/\[bench trace\] step //' | cut -c1-8 | tr '\n' ' '; echo
done
