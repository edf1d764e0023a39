"""Generate golden vectors from the chunkkv REFERENCE itself (run in the build container).

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference cannot travel to the GPU box, so its outputs on seeded inputs are frozen
here as small .npz fixtures that the oracle (tests/test_oracle.py) and the CUDA path
(tests/test_gpu_*.py) are checked against.  Re-running reproduces them bit for bit.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

import chunkkv  # noqa: E402  (reference, from PYTHONPATH)
from chunkkv import kernels as rk  # noqa: E402
from chunkkv import quantizer as rq  # noqa: E402
from chunkkv.attention import AttentionInstance, mixed_decode_attention, reference_attention  # noqa: E402
from chunkkv.harness import RunConfig, synth_workload  # noqa: E402
from chunkkv.attention import prefill_attention  # noqa: E402
from chunkkv.kv_store import build_cache, reconstruct, serialize_cache  # noqa: E402
from chunkkv.toy_model import ToyModel, generate  # noqa: E402
from chunkkv.retrieval import (HashedBowEncoder, TfidfEncoder, build_similarity_report,  # noqa: E402
                               score_chunks, segment_context)
from chunkkv.tiers import Tier  # noqa: E402

TIER_CODE = {Tier.INT2: 0, Tier.INT4: 1, Tier.FP16: 2}


def quantize_cases():
    rng = np.random.default_rng(1234)
    out = {}
    shapes = [(1, 1, 1), (3, 10, 4), (5, 32, 32), (2, 33, 32), (4, 8, 64), (7, 17, 4), (64, 128, 32),
              (33, 7, 32), (10, 100, 32), (16, 128, 32), (1, 3, 3), (6, 16, 16)]
    i = 0
    for rows, cols, gs in shapes:
        for bits in (2, 4):
            x = rng.normal(size=(rows, cols)) * 10.0 ** rng.uniform(-3, 3)
            if i % 5 == 0:
                x[0, :min(cols, gs)] = 3.7  # constant group
            codes, scales, zps = rk.quantize_groups(x, bits, gs)
            packed = rk.pack_codes(codes.reshape(-1), bits)
            out[f"x{i}"] = x
            out[f"meta{i}"] = np.array([rows, cols, gs, bits], np.int64)
            out[f"codes{i}"] = codes
            out[f"scales{i}"] = scales
            out[f"zps{i}"] = zps
            out[f"packed{i}"] = packed
            i += 1
    out["n"] = np.array(i)
    return out


def fp16_rows():
    """fp16-valued D=128 rows incl. adversarial values (exact grid midpoints, subnormals, range ends)."""
    rng = np.random.default_rng(99)
    rows = []
    rows.append(rng.normal(size=(256, 128)))
    rows.append(rng.normal(size=(64, 128)) * 8.0)
    # grid midpoints: lo + (k+0.5)*span/qmax exactly representable in fp16
    mid = np.zeros((32, 128))
    for r in range(32):
        for g in range(4):
            base = np.linspace(-1.0, 1.0, 32)
            base[5] = -1.0 + (0.5 / 3.0) * 2.0
            base[9] = -1.0 + (1.5 / 15.0) * 2.0
            mid[r, 32 * g:32 * g + 32] = base
    rows.append(mid)
    sub = rng.normal(size=(16, 128)) * 1e-6  # fp16 subnormals
    rows.append(sub)
    big = rng.uniform(-60000, 60000, size=(16, 128))
    rows.append(big)
    const = np.full((8, 128), 0.3)
    rows.append(const)
    x = np.concatenate(rows).astype(np.float16)
    xf = x.astype(np.float64)
    out = {"x16": x}
    for bits in (2, 4):
        codes, scales, zps = rk.quantize_groups(xf, bits, 32)
        out[f"codes{bits}"] = codes
        out[f"scales{bits}"] = scales
        out[f"zps{bits}"] = zps
        out[f"packed{bits}"] = rk.pack_codes(codes.reshape(-1), bits)
    return out


def search_cases():
    out = {}
    seeds = [0, 1, 2, 3]
    for s in seeds:
        cfg = RunConfig(context_len=4096, seed=s)
        words, query = synth_workload(cfg)
        cs = segment_context(words, cfg.chunk_size)
        enc = HashedBowEncoder(seed=s)
        chunk_inputs = [" ".join(c) for c in cs.chunks]
        embs = [enc.encode(t) for t in chunk_inputs]
        qe = enc.encode(" ".join(query))
        scores = score_chunks(qe, embs)
        rep = build_similarity_report(scores, cfg.alpha, cfg.beta)
        tiers = np.array([TIER_CODE[t] for t in rep.tiers], np.uint8)
        perm = np.concatenate([np.nonzero(tiers == t)[0] for t in (0, 1, 2)]).astype(np.uint32)
        out[f"emb{s}"] = np.stack([e.vector for e in embs])
        out[f"norm{s}"] = np.array([e.norm for e in embs])
        out[f"q{s}"] = qe.vector
        out[f"qnorm{s}"] = np.array(qe.norm)
        out[f"scores{s}"] = np.array(scores)
        out[f"stats{s}"] = np.array([rep.s_min, rep.s_max, rep.t_low, rep.t_high])
        out[f"tiers{s}"] = tiers
        out[f"perm{s}"] = perm
    out["seeds"] = np.array(seeds)
    return out


def attention_cases():
    out = {}
    rng = np.random.default_rng(7)
    specs = [  # (n_chunks, cs, dim, gs, m, tail, decode)
        (5, 8, 16, 8, 1, 3, 2),
        (8, 32, 64, 32, 4, 0, 0),
        (12, 4, 8, 4, 3, 1, 5),
        (6, 32, 128, 32, 4, 7, 3),
    ]
    for i, (n, cs, d, gs, m, tail, dec) in enumerate(specs):
        tiers = [Tier(t) for t in rng.choice(["int2", "int4", "fp16"], size=n)]
        k = rng.normal(size=(n * cs + tail, d))
        v = rng.normal(size=(n * cs + tail, d))
        cache = build_cache(k, v, tiers, segment_context(list(range(n * cs + tail)), cs), gs)
        kd = rng.normal(size=(dec, d))
        vd = rng.normal(size=(dec, d))
        for r in range(dec):
            cache.append(kd[r], vd[r])
        q = rng.normal(size=(m, d))
        mixed = mixed_decode_attention(AttentionInstance(q=q, cache=cache))
        kr, vr = reconstruct(cache)
        ref = reference_attention(q, kr, vr)
        out[f"spec{i}"] = np.array([n, cs, d, gs, m, tail, dec])
        out[f"tiers{i}"] = np.array([TIER_CODE[t] for t in tiers], np.uint8)
        out[f"k{i}"], out[f"v{i}"], out[f"kd{i}"], out[f"vd{i}"], out[f"q{i}"] = k, v, kd, vd, q
        out[f"mixed{i}"] = mixed
        out[f"ref{i}"] = ref
        out[f"perm{i}"] = cache.perm
        out[f"k_q2_packed{i}"] = cache.k_q2.packed
        out[f"v_q4_scales{i}"] = cache.v_q4.scales
    out["n"] = np.array(len(specs))
    return out


def batched_case():
    """fp16 K/V [L=2, B=2, T, H=2, 128], GQA m=4, per-sequence tier maps from the reference search."""
    rng = np.random.default_rng(2503)
    L, B, H, m, D = 2, 2, 2, 4, 128
    T = 16 * 32 + 7  # 16 chunks + 7-token tail
    k = (rng.normal(size=(L, B, T, H, D))).astype(np.float16)
    v = (rng.normal(size=(L, B, T, H, D))).astype(np.float16)
    k[0, 0, :, 0, 5] *= 8  # outlier channel
    q = (rng.normal(size=(L, B, H * m, D)) * 1.5).astype(np.float16)
    tiers = np.stack([rng.choice([0, 0, 0, 1, 1, 2], size=16).astype(np.uint8) for _ in range(B)])
    tiers[1, :3] = 2
    out = {"k": k, "v": v, "q": q, "tiers": tiers, "dims": np.array([L, B, H, m, T])}
    cs = segment_context(list(range(T)), 32)
    for l in range(L):
        for b in range(B):
            tl = [(Tier.INT2, Tier.INT4, Tier.FP16)[t] for t in tiers[b]]
            for h in range(H):
                cache = build_cache(k[l, b, :, h].astype(np.float64), v[l, b, :, h].astype(np.float64),
                                    tl, cs, 32)
                key = f"{l}_{b}_{h}"
                for name in ("k_q2", "v_q2", "k_q4", "v_q4"):
                    blk = getattr(cache, name)
                    out[f"{name}_packed_{key}"] = blk.packed
                    out[f"{name}_scales_{key}"] = blk.scales
                    out[f"{name}_zps_{key}"] = blk.zero_points
                out[f"perm_{key}"] = cache.perm
                wire = serialize_cache(cache)  # kv_store.py:310-360, the bit-exact wire format
                out[f"wire_len_{key}"] = np.array(len(wire))
                out[f"wire_sha256_{key}"] = np.frombuffer(hashlib.sha256(wire).digest(), np.uint8)
                qq = q[l, b, h * m:(h + 1) * m].astype(np.float64)
                out[f"out_{key}"] = mixed_decode_attention(AttentionInstance(q=qq, cache=cache))
    return out


# toy-model scenarios: (vocab, embed_dim, heads, seed, prompt_len, tier pattern, chunk, group, steps)
TOY_SPECS = [
    (64, 16, 2, 7, 24, "int2_int4", 4, 8, 10),
    (128, 32, 4, 8, 56, "fp16", 8, 8, 16),
    (64, 16, 2, 9, 32, "int4", 8, 8, 4),
    (512, 64, 4, 0, 200, "random", 32, 16, 24),
    (256, 128, 1, 3, 300, "random", 32, 32, 12),
]


def toy_tiers(pattern, n, rng):
    if pattern == "int2_int4":
        return [Tier.INT2, Tier.INT4] * (n // 2) + [Tier.INT2] * (n % 2)
    if pattern in ("fp16", "int4"):
        return [Tier(pattern)] * n
    return [Tier(t) for t in rng.choice(["int2", "int4", "fp16"], size=n)]


def toy_cases():
    """The reference's own caller of the path (toy_model.generate over per-head caches built
    from prefill_attention's K/V), on the tests' scenarios and two larger ones."""
    out = {}
    rng = np.random.default_rng(11)
    for i, (vocab, dim, heads, seed, n_prompt, pattern, cs, gs, steps) in enumerate(TOY_SPECS):
        model = ToyModel(vocab_size=vocab, embed_dim=dim, n_heads=heads, seed=seed)
        prompt = [int(t) for t in rng.integers(0, vocab, size=n_prompt)]
        emb = model.embed(prompt)
        k, v, logits, hidden = prefill_attention(emb, model, return_hidden=True)
        chunk_set = segment_context(prompt, cs)
        tiers = toy_tiers(pattern, chunk_set.n, rng)
        d = model.head_dim
        caches = [build_cache(k[:, h * d:(h + 1) * d], v[:, h * d:(h + 1) * d], tiers, chunk_set, gs)
                  for h in range(heads)]
        first = int(np.argmax(logits))
        gen = generate(model, caches, first, steps, start_pos=n_prompt)
        out[f"spec{i}"] = np.array([vocab, dim, heads, seed, n_prompt, cs, gs, steps])
        out[f"prompt{i}"] = np.array(prompt, np.int64)
        out[f"tiers{i}"] = np.array([TIER_CODE[t] for t in tiers], np.uint8)
        out[f"prefill_logits{i}"] = logits
        out[f"prefill_hidden{i}"] = hidden[-4:]  # last rows (the fixture stays small)
        out[f"first{i}"] = np.array(first)
        out[f"tokens{i}"] = np.array(gen.tokens, np.int64)
        out[f"final_hidden{i}"] = gen.final_hidden
        out[f"w_sum{i}"] = np.array([model.w_e.sum(), model.w_q.sum(), model.w_o.sum()])
    out["n"] = np.array(len(TOY_SPECS))
    return out


def _blob(texts):
    bufs = [t.encode("utf-8") for t in texts]
    off = np.zeros(len(bufs) + 1, np.int64)
    np.cumsum([len(b) for b in bufs], out=off[1:])
    return np.frombuffer(b"".join(bufs) or b"\0", np.uint8).copy(), off


def encoder_cases():
    """HashedBowEncoder / TfidfEncoder on edge-case texts (every str.isspace() separator,
    non-ASCII words, words longer than one 128-byte BLAKE2b block, empty and blank texts, a
    cancelling pair) and on synthetic workloads' chunk texts with their search results."""
    spaces = [c for c in map(chr, range(0x110000)) if c.isspace()]
    rng = np.random.default_rng(31)
    texts = ["", "   ", "\t\n\x0b\x0c\r\x1c", "word", "a b c a", "x" * 128, "y" * 129, "z" * 300 + " q",
             "caf\u00e9 \u4e2d\u6587 \U0001f600 na\u00efve", "a\u00a0b", "\u00a0lead trail\u3000",
             "\u0085\u0085x\u2028y\u2029z"]
    for c in spaces:
        texts.append(f"alpha{c}beta{c}{c}gamma")
    # a word pair landing in the same dim-256 bucket with opposite signs: the bucket cancels
    enc = HashedBowEncoder(seed=0)
    import hashlib
    seen = {}
    for i in range(100000):
        w = f"w{i}"
        h = int.from_bytes(hashlib.blake2b(w.encode(), key=b"0", digest_size=8).digest(), "little")
        b, sgn = h % 256, h >> 63
        if (b, 1 - sgn) in seen:
            texts.append(f"{seen[(b, 1 - sgn)]} {w}")
            break
        seen[(b, sgn)] = w
    for _ in range(40):
        n = int(rng.integers(1, 60))
        texts.append(" ".join(f"w{int(x):05d}" for x in rng.integers(0, 3000, size=n)))
    out = {"spaces": np.array([ord(c) for c in spaces], np.int64)}
    out["text"], out["offsets"] = _blob(texts)
    for seed in (0, 7, 123456789):
        for dim in (256, 100, 1, 4096):
            enc = HashedBowEncoder(dim=dim, seed=seed)
            embs = [enc.encode(t) for t in texts]
            out[f"bow_{seed}_{dim}"] = np.stack([e.vector for e in embs])
            out[f"bow_norm_{seed}_{dim}"] = np.array([e.norm for e in embs])
    tf = TfidfEncoder()
    tf.fit(texts)
    embs = [tf.encode(t) for t in texts]
    out["tfidf"] = np.stack([e.vector for e in embs])
    out["tfidf_norm"] = np.array([e.norm for e in embs])
    # texts -> tiers: the synthetic workloads of search.npz (4K, seeds 0-3) as texts
    for s in (0, 1, 2, 3):
        cfg = RunConfig(context_len=4096, seed=s)
        words, query = synth_workload(cfg)
        cs = segment_context(words, cfg.chunk_size)
        chunk_texts = [" ".join(c) for c in cs.chunks]
        out[f"wl_text{s}"], out[f"wl_offsets{s}"] = _blob(chunk_texts + [" ".join(query)])
    return out


def main():
    assert rk.BACKEND in ("numpy", "compiled")
    np.savez_compressed(os.path.join(HERE, "quantize.npz"), **quantize_cases())
    np.savez_compressed(os.path.join(HERE, "fp16_rows.npz"), **fp16_rows())
    np.savez_compressed(os.path.join(HERE, "search.npz"), **search_cases())
    np.savez_compressed(os.path.join(HERE, "attention.npz"), **attention_cases())
    np.savez_compressed(os.path.join(HERE, "batched.npz"), **batched_case())
    np.savez_compressed(os.path.join(HERE, "toy.npz"), **toy_cases())
    np.savez_compressed(os.path.join(HERE, "encoders.npz"), **encoder_cases())
    print("reference backend:", rk.BACKEND, "chunkkv", chunkkv.__version__, file=sys.stderr)


if __name__ == "__main__":
    main()
