python -m pytest tests/test_gpu_batched.py -m gpu -q -x 2>&1 | tail -1
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-prefill 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ['value','ms_per_step','single_launch_all_layers_gbs']})"
done
timeout 600 python tools/cfg4_bench.py 2>&1 | tail -4
