# grid node blocks 4x4x2 (default now) vs 4x4x4 (bz4 variant): grid timing; grid parity tests
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for lib in "" paper_1305_5179_b200/variants/librbf_bz4.so; do
  timeout 300 python tools/bench_kernels.py --config c4 --iters 10 --ops AUTO ${lib:+--lib $lib} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-default}', d.get('grid_ms'), d.get('grid_nonzero'), {k:round(v['kernel_ms'],3) for k,v in d.items() if k.startswith('op_')})"
done
timeout 1500 python -m pytest tests/test_gpu_hotpath.py tests/test_gpu_fullsize.py tests/test_gpu_mesh.py tests/test_gpu_loopback.py -k "grid or mesh or masked or partition or reconstruct" -x -q > gpurun_out/pytest_g.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_g.log
