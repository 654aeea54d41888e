# final build: full GPU suite + smoke (the suite of sess_r02final.sh ran one build earlier)
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('c4', d['ms_per_step'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['detail']['rel_residual_true'], d['detail']['stage_ms_per_step'])"
