# near-mask fp32 prefilter: zero set / mesh parity + timing
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests/test_gpu_mesh.py tests/test_gpu_solver.py tests/test_gpu_fullsize.py tests/test_gpu_quality.py -k "mesh or zero or quality or masked" -x -q > gpurun_out/pytest_k.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_k.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"near_kernel|near_blocks|data_f32" python tools/prof_grid.py c4 > gpurun_out/near_times.csv 2>&1; echo ncu=$?
grep -E "near|data_f32" gpurun_out/near_times.csv | awk -F'","' '{print $5, $NF}' | cut -c1-60,200-
