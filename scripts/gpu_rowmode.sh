for c in C P B; do for t in 16 32 64 100000; do
line=$(NUMPMP_ROW_MODE_MAX=$t timeout 600 python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -n 1)
python -c "
import json,sys
d=json.loads(sys.argv[1]); r=d['iteration_roofline']
print('$c rowmax=$t', 'ms/it %.4f'%d['ms_per_iteration'], 'k1 %.4f k2 %.4f'%(r['stream_pass_ms'], r['link_pass_ms']))
" "$line"; done; done
