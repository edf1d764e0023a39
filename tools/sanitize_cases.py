"""Small invocations of every kernel for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): search, reorder/quantize/pack, decode (splits 1 and > 1, per-layer PDL chain,
CUDA-graph replay, partials + LSE merge, m = 1 / 4 / 8, exact and precise modes), append,
export, the f64 per-head kernels and the text encoders.  Checks results loosely (the parity
tests do that properly); the point is the sanitizer's verdict."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_23294_b200 import batched, kernels, retrieval  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    dev = torch.device("cuda", 0)
    L, B, H, D, N = 2, 2, 2, 128, 7
    T = N * 32 + 9
    k = torch.from_numpy(rng.normal(size=(L, B, T, H, D)).astype(np.float16)).to(dev)
    v = torch.from_numpy(rng.normal(size=(L, B, T, H, D)).astype(np.float16)).to(dev)
    emb = rng.random(size=(B, N, 64))
    qv = rng.random(size=(B, 64))
    s = retrieval.search_batched(emb, np.linalg.norm(emb, axis=2), qv, np.linalg.norm(qv, axis=1))
    cache = batched.build_cache_batched(k, v, s, decode_capacity=8)
    for m in (1, 4, 8):
        q = torch.from_numpy(rng.normal(size=(L, B, H * m, D)).astype(np.float16)).to(dev)
        for splits in (1, 3):
            out = cache.decode(q, splits=splits)
            for l in range(L):  # per-layer PDL chain
                cache.decode(q[l:l + 1], splits=splits, out=out[l:l + 1], layer=l, pdl=l > 0)
            part = cache.decode_partial(q, splits=splits)
            batched.lse_merge(torch.stack([part, part]))
        # warp-plan schedule: whole batch, per-layer PDL chain, partials
        cache.decode(q, schedule="wp")
        for l in range(L):
            cache.decode(q[l:l + 1], out=out[l:l + 1], layer=l, pdl=l > 0, schedule="wp")
        cache.decode_partial(q, schedule="wp")
    q = torch.from_numpy(rng.normal(size=(L, B, H * 4, D)).astype(np.float16)).to(dev)
    out = torch.empty_like(q)
    g = cache.decode_graph(q, out, splits=2, chains=2)
    g.replay()
    g.replay()
    cache.schedule = "wp"
    g = cache.decode_graph(q, out)
    g.replay()
    g.replay()
    cache.schedule = "auto"
    loop = batched.DecodeLoop(cache, 4, splits=2)
    for _ in range(3):
        loop.step(q, k[:, :, 0], v[:, :, 0])
    cache.export_unit(1, 1, 1)
    # precise and exact decode modes: outlier channels / a huge-scale unit
    k2 = k.clone()
    k2[..., ::32] *= 40
    cache2 = batched.build_cache_batched(k2, v, s)
    cache2.decode(q * 3, splits=2)
    cache2.decode(q * 3, schedule="wp")
    k3 = k.clone()
    k3[0, 0, :, 0, 5] = 30000
    cache3 = batched.build_cache_batched(k3, v, s)
    cache3.decode(q, splits=2)
    cache3.decode(q, schedule="wp")
    # per-head f64 API (kernels facade, quantizer round trip)
    x = rng.normal(size=(40, 70))
    codes, sc, zp = kernels.quantize_groups(x, 4, 32)
    packed = kernels.pack_codes(codes.reshape(-1), 4)
    kernels.unpack_codes(packed, 4, codes.size)
    kernels.matmul_packed(rng.normal(size=(3, 70)), packed, sc, zp, 40, 70, 4, 32, True)
    # text encoders + search from text
    texts = [["alpha beta gamma", "delta  epsilon\tzeta", "", "eta theta iota kappa"]]
    retrieval.search_texts(texts, ["beta gamma delta"], 0.6, 0.1, retrieval.HashedBowEncoder(seed=0),
                           check=False)
    torch.cuda.synchronize()
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
