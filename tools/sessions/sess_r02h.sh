# symmetric-kernel variants: default (KB store pinned + asm shfl) vs kb0 (predicated KB store) vs sh0 (intrinsic shfl)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for lib in "" paper_1305_5179_b200/variants/librbf_kb0.so paper_1305_5179_b200/variants/librbf_sh0.so ""; do
  timeout 300 python tools/bench_kernels.py --config c4 --iters 20 --no-grid --ops SYM_WIDE ${lib:+--lib $lib} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-default}', {k: (round(v['kernel_ms'],4), round(v['frac_mufu'],4), '%.1e'%v['max_err_over_g']) for k,v in d.items() if k.startswith('op_')})"
done
