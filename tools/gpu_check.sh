# quick GPU check: build, GPU suite (excluding the slow full-size module unless FULL=1), smoke, short bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
if [ "${FULL:-0}" = 1 ]; then SEL="gpu"; else SEL="gpu and not slow"; fi
timeout ${PYT:-1500} python -m pytest tests -m "$SEL" -x -q ${PYARGS:-} > gpurun_out/pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 ${BENCHARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('ms/step', round(d['ms_per_step'],2), 'value %.3e'%d['value'], 'frac', round(d['roofline']['frac'],4), 'mv ms', round(d['roofline']['avg_launch_ms'],4), 'res', d['detail']['rel_residual_true'], d['detail']['stage_ms_per_step'])
" 2>&1 | tail -2
