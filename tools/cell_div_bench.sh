# whole-step effect of the cell edge (and the wide-plan span) at c4
for v in "3.999 4" "2.999 2" "2.999 3" "2.499 2"; do set -- $v
RBF_BENCH_CELL_DIV=$1 RBF_WIDE_SPAN=$2 timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['detail']['stage_ms_per_step']
print('div $1 span $2', round(d['ms_per_step'],1), 'res', '%.3e' % d['detail']['rel_residual_true'], {k: round(v,1) for k,v in s.items()}, 'blocks', d['detail']['ras_blocks'])"
done
