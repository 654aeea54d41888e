# round-2 verification session: build, full GPU suite, smoke, bench, launch list, ncu of grid + cell build kernels
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e > gpurun_out/ncu.log 2>&1; echo ncu=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sum_f32_kernel|mark_node_blocks|radix_scatter|gather_sorted|radix_hist|sum_f32_symb" -c 12 -o gpurun_out/grid_cells_full python tools/prof_step.py c4 > gpurun_out/ncu_gc.log 2>&1; echo ncu_gc=$?
