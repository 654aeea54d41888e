# c3 / c5 bench lines with the current library, and the fp64 symmetric kernel's instruction mix
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench_c3=$?
python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print('c3', d['ms_per_step'], d['roofline']['frac'], d['detail']['rel_residual_true'], d['detail']['stage_ms_per_step'])"
timeout 1500 python bench.py --config c5 --steps 2 --warmup 3 --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench_c5=$?
python -c "import json; d=json.load(open('gpurun_out/bench_c5.json')); print('c5', d['ms_per_step'], d['roofline']['frac'], d['detail']['rel_residual_true'], d['detail']['stage_ms_per_step'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sum_f64_sym" -c 1 -o gpurun_out/f64sym python tools/prof_step.py c4 > gpurun_out/ncu_f64.log 2>&1; echo ncu=$?
ncu -i gpurun_out/f64sym.ncu-rep --page source --csv --print-source sass > gpurun_out/f64sym_sass.csv 2>/dev/null; echo src=$?
