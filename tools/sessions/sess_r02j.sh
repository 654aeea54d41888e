# apply blocks-per-CTA variants + ncu of the near kernel
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for lib in "" paper_1305_5179_b200/variants/librbf_ap2.so paper_1305_5179_b200/variants/librbf_ap4.so; do
  timeout 300 python tools/bench_kernels.py --config c4 --iters 20 --no-grid --ops AUTO --precond ${lib:+--lib $lib} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-default}', d.get('precond_setup_ms'), d.get('precond_apply_ms'))"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"near_kernel" -c 1 -o gpurun_out/near_full python tools/prof_grid.py c4 > gpurun_out/ncu_near.log 2>&1; echo ncu=$?
