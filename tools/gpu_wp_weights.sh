for rep in 1 2; do for w in ${WS:-1.06,2.0 1.2,3.0 1.3,2.0 1.4,2.0 1.3,3.0 1.2,4.0}; do
CKV_WP_W=$w timeout 600 python bench.py --chains 1 --steps 20 --warmup 5 --no-cpu-baseline --no-prefill --no-tpot --no-sustained 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('w $w', d['value'], d['ms_per_step'], d['single_launch_all_layers_gbs'], d['clocks']['reasons'])"
done; done
