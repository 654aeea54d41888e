# mesh tests (c1 + analytic + c4/c3 crop), then compute-sanitizer racecheck / synccheck / memcheck on the small workload
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_mesh.py tests/test_gpu_fullsize.py -k "mesh" -x -q > gpurun_out/pytest_mesh.log 2>&1; echo pytest_mesh=$?; tail -3 gpurun_out/pytest_mesh.log
timeout 300 python tools/sanitize_run.py --small > gpurun_out/san_plain.log 2>&1; echo plain=$?; tail -1 gpurun_out/san_plain.log
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 --log-file gpurun_out/san_$tool.txt python tools/sanitize_run.py --small > gpurun_out/san_$tool.log 2>&1; echo $tool=$?; tail -2 gpurun_out/san_$tool.txt
done
