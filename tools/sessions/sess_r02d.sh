# full GPU suite + bench (tight grid marking, near-mask block prefilter, batched block-Jacobi apply)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_all.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['ms_per_step'], d['roofline']['frac'], d['detail']['isosurface'], d['detail']['stage_ms_per_step'], d['detail']['visited_pairs_grid'])"
