# mesh tests (c1 + analytic + c4/c3 crop), bench with the isosurface report, ncu of the grid path
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_mesh.py tests/test_gpu_fullsize.py -k "mesh" -x -q > gpurun_out/pytest_mesh.log 2>&1; echo pytest_mesh=$?; tail -3 gpurun_out/pytest_mesh.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['ms_per_step'], d['detail']['isosurface'], d['detail']['stage_ms_per_step'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sum_f32_kernel|mark_node_blocks|near_kernel|mt_|mark_near" -c 12 -o gpurun_out/grid_full python tools/prof_grid.py c4 > gpurun_out/ncu_grid.log 2>&1; echo ncu_grid=$?
