"""CPU, world_size 2 over gloo: the split-KV exchange of (acc, m, l) partials and the LSE merge
reproduce single-rank attention (the NCCL path runs the same code with CUDA tensors)."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ckv_oracle as O
from paper_2503_23294_b200.distributed import exchange_partials, sequence_shard_plan


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, k, v, tiers, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cache = O.build_cache(k, v, tiers, 32, 32)
        perm, counts = O.stable_perm(tiers)
        plan, owns_tail = sequence_shard_plan(counts[None], world, rank)
        a2, b2, a4, b4, af, bf = plan[0]
        # this rank's rows in the reordered sequence (INT2 || INT4 || FP16 chunks || tail)
        kr, vr = O.reconstruct(cache)
        order = O.token_order(cache)
        rows = np.concatenate([np.arange(a2 * 32, b2 * 32), np.arange(a4 * 32, b4 * 32),
                               np.arange(af * 32, bf * 32)])
        if owns_tail:
            rows = np.concatenate([rows, np.arange(counts.sum() * 32, k.shape[0])])
        kk, vv = kr[order[rows]], vr[order[rows]]
        s = (q @ kk.T) / np.sqrt(q.shape[1]) / np.log(2.0)  # log2 domain
        m = s.max(axis=1) if s.shape[1] else np.full(q.shape[0], -np.inf)
        p = np.exp2(s - m[:, None]) if s.shape[1] else np.zeros((q.shape[0], 0))
        part = np.concatenate([p @ vv if s.shape[1] else np.zeros((q.shape[0], vv.shape[1])),
                               m[:, None], p.sum(axis=1)[:, None]], axis=1)
        gathered = exchange_partials(torch.from_numpy(part.astype(np.float32)))
        g = gathered.numpy().astype(np.float64)
        d = q.shape[1]
        out = O.lse_merge(g[:, :, d], g[:, :, d + 1], g[:, :, :d])
        if rank == 0:
            np.save(result_path, out)
    finally:
        dist.destroy_process_group()


def test_split_kv_exchange_world2(tmp_path):
    rng = np.random.default_rng(3)
    n, d, m = 12, 32, 4
    T = n * 32 + 5
    k, v = rng.normal(size=(T, d)), rng.normal(size=(T, d))
    q = rng.normal(size=(m, d))
    tiers = rng.choice([0, 1, 2], size=n).astype(np.uint8)
    path = str(tmp_path / "out.npy")
    mp.spawn(_worker, args=(2, _free_port(), q, k, v, tiers, path), nprocs=2, join=True)
    got = np.load(path)
    cache = O.build_cache(k, v, tiers, 32, 32)
    want = O.reference_attention(q, *O.reconstruct(cache))
    assert np.max(np.abs(got - want)) < 1e-5  # f32 partials


def test_layer_and_batch_shards_partition():
    from paper_2503_23294_b200.distributed import batch_shard, layer_shard

    for n in (1, 7, 32, 40, 64):
        for world in (1, 2, 3, 4, 8):
            for fn in (layer_shard, batch_shard):
                parts = [fn(n, world, r) for r in range(world)]
                assert parts[0][0] == 0 and parts[-1][1] == n
                assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
                assert max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1
