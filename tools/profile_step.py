"""One eager bench step of a BASELINE config between cudaProfilerStart/Stop, for
`ncu --profile-from-start off` (launch lists and full captures of exactly one
batch; tools/gpu_prof_r2.sh).  Uniform-random key/query material (all kernels
are data-oblivious), records generated on the GPU.

  python tools/profile_step.py --config 3
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    args = ap.parse_args()
    import torch

    import bench
    import paper_2604_04696_b200 as G
    from paper_2604_04696_b200 import _native as nat

    d0, d1, B, rb, pb, _ = bench.CONFIGS[args.config]
    params = G.HeParams(G.default_basis(4096), pb)
    cfg = G.DbConfig(d0, d1, rb)
    recs = bench._device_records(torch, cfg.records, rb, 0, 1)
    db = G.encode_database_device(recs, cfg, params, compact=args.config >= 4)
    del recs
    ctx = db.ctx
    ns = argparse.Namespace(material="uniform", clients="distinct")
    q, slots = bench._client_material(G, ctx, params, d0, d1, B, np.random.default_rng(1), ns, ctx.lib, nat)
    nat.check(ctx.lib.gpir_set_graphs(ctx.h, 0), "graphs off")
    d_q = torch.from_numpy(q.view(np.int32).reshape(-1)).cuda()
    d_o = torch.empty_like(d_q)

    def step():
        nat.check(ctx.lib.gpir_answer_batch_dev(ctx.h, db.handle, C.c_void_p(d_q.data_ptr()),
                                                nat.ptr(slots, C.c_int32), B, None, 0, None, 0,
                                                C.c_void_p(d_o.data_ptr()), None, None), "answer")

    step()  # lazy allocations and byte-plane packing outside the profiled range
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    step()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("profiled one step of config", args.config)


if __name__ == "__main__":
    main()
