"""cfg5 prefill (search + reorder/quantize/pack, 128K x 32 layers x 8 kv heads) alone: the
bench.py prefill sub-object, for quick iterations on the quantize kernel."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402

if __name__ == "__main__":
    torch.cuda.set_device(0)
    print(json.dumps(bench.bench_prefill(torch, torch.device("cuda", 0), steps=5)))
