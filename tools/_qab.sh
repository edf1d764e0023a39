python -m pytest tests -q -x -m gpu -k "batched or cfg5 or api or adversarial or fused or quantize" 2>&1 | tail -1
for i in 1 2; do timeout 300 python tools/prefill_bench.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['quantize_ms'])"; done
bash tools/gpu_ncu_quant.sh 2>&1 | grep -E "bank_conflicts|inst_executed.sum|duration"
