import sys, numpy as np, torch, time
sys.path.insert(0, '/root/repo')
import __graft_entry__ as ge
ge.smoke()
from oracle import ckv_oracle as O
from paper_2503_23294_b200 import batched, retrieval, quantizer, kernels
# per-head quick checks
x = np.random.default_rng(1).normal(size=(7,17))
blk = quantizer.quantize(x, 2, 4)
ob = O.quantize(x, 2, 4)
print("quantize f64 exact:", np.array_equal(blk.packed, ob.packed), np.array_equal(blk.scales, ob.scales))
# decode splits consistency, all tiers, slow path, m=1,8
rng = np.random.default_rng(5)
dev='cuda'
for (m, tiers_kind, scale) in [(4,'mix',1.0),(1,'mix',1.0),(8,'mix',1.0),(4,'int2',1.0),(4,'int4',1.0),(4,'fp16',1.0),(4,'mix',300.0)]:
    L,B,H,D=2,3,2,128
    T=20*32+9
    k=torch.from_numpy((rng.normal(size=(L,B,T,H,D))*scale).astype(np.float16)).to(dev)
    v=torch.from_numpy((rng.normal(size=(L,B,T,H,D))*scale).astype(np.float16)).to(dev)
    q=torch.from_numpy((rng.normal(size=(L,B,H*m,D))/scale).astype(np.float16)).to(dev)
    if tiers_kind=='mix': tiers=rng.choice([0,0,1,2],size=(B,20)).astype(np.uint8)
    else: tiers=np.full((B,20),{'int2':0,'int4':1,'fp16':2}[tiers_kind],np.uint8)
    thr=np.array([[0.5,1.5]]*B)
    s=retrieval.assign_tiers_batched(tiers.astype(np.float64), thr)
    cache=batched.build_cache_batched(k,v,s)
    outs=[cache.decode(q,splits=sp).float().cpu().numpy() for sp in (1,3,7)]
    kh,vh,qh=k.cpu().numpy(),v.cpu().numpy(),q.cpu().numpy()
    worst=0; wrel=0
    for l in range(L):
      for b in range(B):
        for h in range(H):
          oc=O.build_cache(kh[l,b,:,h].astype(np.float64),vh[l,b,:,h].astype(np.float64),tiers[b],32,32)
          ex=cache.export_unit(l,b,h)
          assert np.array_equal(ex.k_q2.packed, oc.k_q2.packed) and np.array_equal(ex.v_q2.packed, oc.v_q2.packed)
          assert np.array_equal(ex.k_q4.packed, oc.k_q4.packed) and np.array_equal(ex.v_q4.scales, oc.v_q4.scales)
          ref=O.mixed_decode_attention(qh[l,b,h*m:(h+1)*m].astype(np.float64),oc)
          for o in outs:
            e=np.max(np.abs(o[l,b,h*m:(h+1)*m]-ref)); worst=max(worst,e); wrel=max(wrel,e/np.max(np.abs(ref)))
    print(f"m={m} {tiers_kind} scale={scale}: max abs err {worst:.3e} rel {wrel:.3e}")
