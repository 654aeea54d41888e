Q="index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
for ms in 200 1000; do
nvidia-smi -i 0 --query-gpu=$Q --format=csv,noheader,nounits -lms $ms > /dev/null 2>&1 & NP=$!; sleep 1
echo "lms=$ms"; timeout 400 python tools/step_trace.py c4 6 2>&1 | tail -6 | python -c "
import json,sys
print([json.loads(l)['wall_ms'] for l in sys.stdin])"
kill $NP; sleep 1
done
echo "none"; timeout 400 python tools/step_trace.py c4 6 2>&1 | tail -6 | python -c "
import json,sys
print([json.loads(l)['wall_ms'] for l in sys.stdin])"
