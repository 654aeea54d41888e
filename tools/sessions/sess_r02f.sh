# GJ warp-count variants (precond setup/apply timing at c4) + near-kernel timing
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for lib in "" paper_1305_5179_b200/variants/librbf_gjA.so paper_1305_5179_b200/variants/librbf_gjB.so; do
  timeout 300 python tools/bench_kernels.py --config c4 --iters 10 --no-grid --ops AUTO --precond ${lib:+--lib $lib} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-default}', d.get('precond_setup_ms'), d.get('precond_apply_ms'))"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"near_kernel|near_blocks|sum_f32_kernel|mt_" python tools/prof_grid.py c4 > gpurun_out/near_times.csv 2>&1; echo ncu=$?
grep -E "near|sum_f32|mt_" gpurun_out/near_times.csv | awk -F'","' '{print $5, $NF}' | head -20
