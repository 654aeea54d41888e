# is the nvidia-smi sampler stretching the host-paced stages of the device-timed loop? (cells stage 1.7 .. 17 ms between runs; the e2e loop, which runs without the sampler, never moved)
for mode in default noclocks lms1000 default2; do
  case $mode in
    noclocks) export RBF_BENCH_NO_CLOCKS=1;;
    lms1000) unset RBF_BENCH_NO_CLOCKS; export RBF_BENCH_CLOCKS_MS=1000;;
    *) unset RBF_BENCH_NO_CLOCKS; unset RBF_BENCH_CLOCKS_MS;;
  esac
  RBF_BENCH_TRACE=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_$mode.json 2> gpurun_out/bench_$mode.err; echo bench=$?
  python -c "import json; d=json.load(open('gpurun_out/bench_$mode.json')); print('$mode', d['ms_per_step'], d['clocks'].get('samples'), d['detail']['stage_ms_per_step'])"
  grep "bench trace" gpurun_out/bench_$mode.err | tr '\n' ';' | cut -c1-600; echo
done
