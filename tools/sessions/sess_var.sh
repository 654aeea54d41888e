# run bench_kernels (solver operator timings) for the default library and each variant .so
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for lib in "" $(ls paper_1305_5179_b200/variants/*.so 2>/dev/null); do
  timeout 300 python tools/bench_kernels.py --config ${CFG:-c4} --iters 20 --no-grid --ops ${OPS:-SYM_WIDE} ${lib:+--lib $lib} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-default}', {k: (round(v['kernel_ms'],4), round(v['frac_mufu'],4), '%.1e'%v['max_err_over_g']) for k,v in d.items() if k.startswith('op_')})"
done
