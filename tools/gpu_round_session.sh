# full round check on one B200: build, GPU suite, smoke, bench, launch list, ncu of the top kernels
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e > gpurun_out/ncu.log 2>&1; echo ncu=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sum_f32_symw -s 1 -c 1 -o gpurun_out/symw_full python tools/prof_step.py > gpurun_out/ncu_symw.log 2>&1; echo ncu_symw=$?
timeout 600 ncu --set full --clock-control none -k regex:"sum_f64_sym|apply_sym|gj_inverse" -c 3 -o gpurun_out/others_full python tools/prof_step.py > gpurun_out/ncu_others.log 2>&1; echo ncu_others=$?
