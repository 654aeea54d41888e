python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sum_f32_symb -s 2 -c 1 -o gpurun_out/symb_r02a python tools/prof_step.py c4 > gpurun_out/ncu_symb.log 2>&1; echo ncu=$?
