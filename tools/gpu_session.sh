python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python tools/sweep_tiles.py c4 2>&1 | sed -n 2,3p
timeout 300 python tools/bench_kernels.py --config c4 --iters 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('matvec', d['matvec_f32_ms'], 'grid', d['grid_ms'])"
