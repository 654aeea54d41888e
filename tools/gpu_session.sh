python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
nproc
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log; tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 2 --warmup 1 > gpurun_out/bench_try.json 2> gpurun_out/bench_try.err; tail -3 gpurun_out/bench_try.err; cat gpurun_out/bench_try.json
