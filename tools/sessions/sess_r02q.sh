# source-level attribution of the dominant kernel (symmetric fp32, c4)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python tools/prof_step.py c4 > gpurun_out/prof_plain.log 2>&1; echo plain=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sum_f32_symb -s 1 -c 1 -o gpurun_out/symb_src python tools/prof_step.py c4 > gpurun_out/ncu_symb.log 2>&1; echo ncu=$?
ncu -i gpurun_out/symb_src.ncu-rep --page source --csv --print-source sass > gpurun_out/symb_sass.csv 2>/dev/null; echo sass=$?
ncu -i gpurun_out/symb_src.ncu-rep --page source --csv --print-source cuda > gpurun_out/symb_cuda.csv 2>/dev/null; echo cuda=$?
ncu -i gpurun_out/symb_src.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/symb_cudasass.csv 2>/dev/null; echo cudasass=$?
ncu -i gpurun_out/symb_src.ncu-rep --page raw --csv > gpurun_out/symb_raw.csv 2>/dev/null; echo raw=$?
ls -la gpurun_out/
