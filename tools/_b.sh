python -m pytest tests -q -x -m gpu > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-prefill 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ['value','eager_launches_gbs','single_launch_all_layers_gbs']}, d['e2e']['value'])"; done
timeout 600 python tools/cfg4_bench.py 2>&1 | tail -3
