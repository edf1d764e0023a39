"""Small invocations of every kernel for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): search, reorder/quantize/pack, decode (splits 1 and > 1, per-layer PDL chain,
CUDA-graph replay, micro-batch chains (sequence and kv-head ranges) on the split kernel and on the warp plan, partials + LSE
merge by array and by pointers, m = 1 / 4 / 8, outlier-K and huge-scale units), append, export,
the tile-native reconstruct, the f64 per-head kernels and the text encoders.  Checks results loosely (the parity
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
    g = cache.decode_graph(q, out, splits=cache.chain_splits(4), chains=B)  # the bench's default step
    g.replay()
    g.replay()
    g = cache.decode_graph(q, out, splits=3, chains=B * H)  # chains over (sequence, kv-head range)
    g.replay()
    g.replay()
    for h in range(H):  # split-KV partials of one kv-head range each (cfg3's head chains)
        for l in range(L):
            cache.decode_partial(q[l:l + 1], splits=2, layer=l, pdl=l > 0, heads=(h, h + 1))
    for b in range(B):  # warp plan over sequence ranges
        for l in range(L):
            cache.decode(q[l:l + 1], out=out[l:l + 1], layer=l, pdl=l > 0, seqs=(b, b + 1), schedule="wp")
    # LSE merge through a device array of partial-buffer pointers (the peer-memory exchange's merge)
    from paper_2503_23294_b200 import _lib
    pa, pb = cache.decode_partial(q, splits=2), cache.decode_partial(q, splits=3)
    ptrs = torch.tensor([pa.data_ptr(), pb.data_ptr()], dtype=torch.int64, device=dev)
    merged = torch.empty((pa.shape[0], D), dtype=torch.float16, device=dev)
    _lib.call("ckv_lse_merge_ptrs", _lib.ptr(ptrs), 2, pa.shape[0], _lib.ptr(merged), _lib.stream())
    cache.reconstruct()
    loop = batched.DecodeLoop(cache, 4, splits=2)
    for _ in range(3):
        loop.step(q, k[:, :, 0], v[:, :, 0])
    cache.export_unit(1, 1, 1)
    # outlier channels (wide K groups) / a huge-scale unit
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
