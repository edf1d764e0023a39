mkdir -p gpurun_out
./tools/subnormal_probe 2>&1 | tee gpurun_out/subnormal.txt
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-prefill --no-tpot 2>/dev/null | tail -1 > gpurun_out/b0.json
python -c "import json; d=json.load(open('gpurun_out/b0.json')); print(d['value'], d['roofline'], d['single_launch_all_layers_gbs'], d['clocks'])"
timeout 300 python tools/wp_timeline.py 2>&1 | tail -16
