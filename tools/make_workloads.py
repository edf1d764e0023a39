"""Freeze the benchmark workloads' search inputs from the chunkkv REFERENCE (build container only).

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python tools/make_workloads.py

For each synthetic (context, query) of BASELINE.json's configs (harness.synth_workload at the
paper operating point alpha=0.6, beta=0.1, chunk 32, hashed-BoW encoder) this stores the chunk
and query embeddings (the GPU search kernel's inputs) plus the reference's own tier map, so the
bench can run Module I on the device and assert the tier maps match the reference at full size.
Embeddings are stored sparsely (<= 32 nonzeros per 256-d BoW vector).
"""

import os

import numpy as np

from chunkkv.harness import RunConfig, synth_workload
from chunkkv.retrieval import HashedBowEncoder, build_similarity_report, score_chunks, segment_context
from chunkkv.tiers import Tier

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "workloads.npz")
CODE = {Tier.INT2: 0, Tier.INT4: 1, Tier.FP16: 2}


def one(ctx, seed):
    cfg = RunConfig(context_len=ctx, seed=seed)
    words, query = synth_workload(cfg)
    cs = segment_context(words, cfg.chunk_size)
    enc = HashedBowEncoder(seed=seed)
    embs = [enc.encode(" ".join(c)) for c in cs.chunks]
    qe = enc.encode(" ".join(query))
    scores = score_chunks(qe, embs)
    rep = build_similarity_report(scores, cfg.alpha, cfg.beta)
    dense = np.stack([e.vector for e in embs])
    nz = max(int((dense != 0).sum(axis=1).max()), 1)
    idx = np.zeros((dense.shape[0], nz), np.uint8)
    val = np.zeros((dense.shape[0], nz), np.float64)
    for i, row in enumerate(dense):
        j = np.nonzero(row)[0]
        idx[i, :j.size] = j
        val[i, :j.size] = row[j]
    return dict(idx=idx, val=val, norm=np.array([e.norm for e in embs]), q=qe.vector,
                qnorm=np.array(qe.norm), tiers=np.array([CODE[t] for t in rep.tiers], np.uint8),
                stats=np.array([rep.s_min, rep.s_max, rep.t_low, rep.t_high]))


def main():
    out = {}
    for ctx, seeds in ((32768, range(8)), (131072, range(1)), (16384, range(8)), (4096, range(1))):
        for s in seeds:
            for k, v in one(ctx, s).items():
                out[f"{ctx}_{s}_{k}"] = v
    np.savez_compressed(OUT, **out)
    print(OUT, os.path.getsize(OUT))


if __name__ == "__main__":
    main()
