python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python tools/bench_kernels.py --config c4 --iters 20 > gpurun_out/bk.json 2> gpurun_out/bk.err; echo bk=$?; cat gpurun_out/bk.json; tail -3 gpurun_out/bk.err
