# re-measure the c4 line (two runs) after the final2 anomaly (cells stage 7.3 ms, step 186 ms while e2e stayed at 173.5 ms)
for i in 1 2; do
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench_$i.json')); print('c4', d['ms_per_step'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['detail']['rel_residual_true'], d['detail']['stage_ms_per_step'], d['config']['l2'])"
done
