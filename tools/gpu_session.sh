python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_solver.py -q -x 2>&1 | tail -3
timeout 600 python tools/prof_precond.py c4 2>&1 | tail -1
timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e 2>gpurun_out/bench5.err > gpurun_out/bench5.json; python -c "import json; d=json.load(open('gpurun_out/bench5.json')); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['detail']['stage_ms_per_step'])"
