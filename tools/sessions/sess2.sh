python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_full.log 2>&1; echo pytest_full=$?; tail -3 gpurun_out/pytest_full.log
timeout 600 python tools/c4_long_solve.py --iters 1000 > gpurun_out/c4_long.json 2> gpurun_out/c4_long.err; echo long=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sum_f32_symw -s 2 -c 1 -o gpurun_out/symw_r02a python tools/prof_step.py c4 > gpurun_out/ncu_symw.log 2>&1; echo ncu=$?
