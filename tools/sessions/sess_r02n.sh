# apply staging-cap variants (setup/apply timing at c4)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for lib in "" paper_1305_5179_b200/variants/librbf_c1.so paper_1305_5179_b200/variants/librbf_c2.so paper_1305_5179_b200/variants/librbf_c3.so; do
  timeout 300 python tools/bench_kernels.py --config c4 --iters 20 --no-grid --ops AUTO --precond ${lib:+--lib $lib} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-default}', d.get('precond_setup_ms'), d.get('precond_apply_ms'))"
done
