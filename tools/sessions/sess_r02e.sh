# full GPU suite (incl. race probe with the checked build), bench, ncu of the setup/apply/Krylov kernels
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
python -m paper_1305_5179_b200.build --checked > gpurun_out/build_checked.log 2>&1; echo build_checked=$?
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_all.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['ms_per_step'], d['roofline']['frac'], d['detail']['stage_ms_per_step'], d['detail']['rel_residual_true'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e > gpurun_out/ncu.log 2>&1; echo ncu=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gj_spd|apply_sym|multi_axpy|multi_dot" -c 8 -o gpurun_out/setup_full python tools/prof_step.py c4 > gpurun_out/ncu_setup.log 2>&1; echo ncu_setup=$?
