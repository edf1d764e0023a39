for i in 1 2; do timeout 300 python tools/prefill_bench.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['quantize_ms'])"; done
bash tools/gpu_ncu_quant.sh 2>&1 | grep -E "inst_executed.sum|duration|issue_active|dram__bytes"
