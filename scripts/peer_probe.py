"""Debug probe for NALAR_COLL_PEER with in-process ranks: host time of each call."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from nalar_gen import c2
from paper_2601_05109_b200 import nalar
from paper_2601_05109_b200.sharding import connect_local, shard_bounds

s = c2(2)
G = 2
flags = nalar.NALAR_F_NO_GRAPH if "--nograph" in sys.argv else 0
streams = [torch.cuda.Stream() for _ in range(G)]
print("stream flags query:", [torch.cuda.current_stream().cuda_stream], flush=True)
ctxs, shards = [], []
for k, (w0, w1) in enumerate(shard_bounds(s.wf_fut_off, G)):
    ctxs.append(nalar.Context.for_snapshot(s, world=G, rank=k, collective=nalar.NALAR_COLL_PEER,
                                           stream=streams[k].cuda_stream if "--own" not in sys.argv else None, flags=flags))
    shards.append(s.slice_workflows(w0, w1))
connect_local(ctxs)
for c, sh in zip(ctxs, shards):
    c.upload(sh)
for e in range(3):
    for k, c in enumerate(ctxs):
        t0 = time.time(); c.epoch("srtf"); print(f"epoch {e} rank {k}: {1e3*(time.time()-t0):.2f} ms", flush=True)
for k, c in enumerate(ctxs):
    t0 = time.time()
    try:
        c.fetch(); print(f"fetch {k} ok {1e3*(time.time()-t0):.1f} ms", flush=True)
    except Exception as ex:
        print(f"fetch {k} failed {1e3*(time.time()-t0):.1f} ms: {ex}", flush=True)
