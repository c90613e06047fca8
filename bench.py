"""GPIR server-pipeline benchmark (BASELINE.json metric: PIR queries/sec, batched).

One step = one full batch through the server pipeline (ExpandQuery -> RGSW
assembly -> RowSel -> ColTor) for B client queries against the encoded DB.
Default workload = BASELINE configs[1]: 1 GiB encoded DB (D0=256 x D1=64
polys, 8 KiB records at P=2^16), batch of 32 distinct clients, one B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 1|2|3]

`value` is device-timed QPS with queries resident in HBM; `e2e` is the same
metric through the C ABI host entry point `gpir_answer_batch` with pinned
host buffers (H2D of queries + D2H of responses inside the timed region).
`--impl reference` times the CPU oracle port of the reference's answer_batch
on this host (rank 0 only).  Multi-GPU (torchrun, one rank per GPU): each
rank serves its own batch against its own copy of the DB shard (see
DESIGN.md "Multi-GPU"); QPS is summed over ranks with max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(ROOT, ".numba_cache"))

CONFIGS = {
    # name: (d0, d1, B, record_bytes, plain_bits, description)
    1: (16, 16, 1, 16384, 32, "config1: 16 MiB encoded DB (16x16, 16 KiB records, P=2^32), 1 query"),
    2: (256, 64, 32, 8192, 16, "config2: 1 GiB encoded DB (256x64 polys, 8 KiB records, P=2^16), batch 32 clients"),
    3: (256, 512, 128, 8192, 16, "config3: 8 GiB encoded DB (256x512 polys, 8 KiB records, P=2^16), batch 128 clients"),
}


def config_of(args):
    """The BASELINE config, with the batch overridden by --batch (a sweep at the same DB geometry)."""
    d0, d1, B, rb, pb, desc = CONFIGS[args.config]
    if getattr(args, "batch", 0):
        desc = f"{desc.split(', batch')[0]}, batch {args.batch} (sweep; the config's own batch is {B})"
        B = args.batch
    return d0, d1, B, rb, pb, desc


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled (NVML, every 5 ms) during the timed region."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.sm, self.mx, self.reasons = [], None, set()
        self._stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def loop():
                while True:
                    self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.reasons.update(k for k, m in self.REASONS.items() if r & m)
                    if self._stop.wait(0.005):
                        return

            self.t = threading.Thread(target=loop, daemon=True)
            self.t.start()
        except Exception as e:  # no NVML: report the gap instead of a number
            self.err = str(e)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.t is not None:
            self.t.join(timeout=2)

    def summary(self):
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None, "sm_max_mhz": self.mx,
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


def ncu_traffic(prefix="k_rowsel_tc"):
    """dram read+write bytes per launch of the RowSel kernel from the newest committed
    `ncu --set full` summary (profiles/*_ncu.json, tools/ncu_summary.py), or None."""
    import glob

    best = None
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu.json")), key=os.path.getmtime):
        try:
            js = json.load(open(f))
        except Exception:
            continue
        for k, d in js.get("kernels", {}).items():
            if k.startswith(prefix) and "traffic_bytes" in d:
                best = (d["traffic_bytes"], os.path.basename(f), k)
    return best


def dominant_kernel():
    """The largest-share kernel of the newest committed ncu launch list (one config-2
    bench step, profiles/*_ncu.json) with its pipe counters from the full capture:
    the kernel `roofline` (RowSel, the north star's roofline target) is not."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu.json")), key=os.path.getmtime)
    for f in reversed(files):
        try:
            js = json.load(open(f))
        except Exception:
            continue
        ll = js.get("launch_list") or {}
        if not ll:
            continue
        tot = sum(v["ns"] for v in ll.values())
        name, v = max(ll.items(), key=lambda kv: kv[1]["ns"])
        full = js.get("kernels", {}).get(name, {})

        def pct(key):
            m = full.get(key)
            return float(m["value"]) / 100 if isinstance(m, dict) else None

        return {"kernel": name, "share_of_launch_list": v["ns"] / tot,
                "bound": "FMA-heavy integer pipe (IMAD, IMAD.HI)",
                "fmaheavy_busy": pct("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                "issue_active": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                "phase_floor_frac": "see phase_roofline.ExpandQuery (live)",
                "src": f"profiles/{os.path.basename(f)} (ncu launch list + --set full)"}
    return None


def phase_rooflines(d0, d1, B, k, n, ell, phases, rs_bytes, hbm_gbs, sms=148, clk_hz=1.965e9):
    """Per-phase roofline fractions.  The tree phases (ExpandQuery, RGSW
    assembly, ColTor) are bound by the FMA-heavy integer pipe: a Shoup
    butterfly is one IMAD.HI (quarter rate) + two IMADs (half rate) = 8
    SMSP-cycles per warp, an exact 64-bit MAC one IMAD.WIDE = 4 (measured,
    tools/micro/pipes.cu).  Algorithmic work per node / external product, with
    the top gadget digit folded into the keys: ExpandQuery node =
    k iNTTs + k (ell-1) digit NTTs, 2 k ell n MACs; external product = 2 k iNTTs
    + 2 k (ell-1) digit NTTs, 4 k ell n MACs.  RowSel is bound by HBM."""
    bfly = (n // 2) * (n.bit_length() - 1)
    total = d0 + (d1.bit_length() - 1) * ell
    stages = (total - 1).bit_length()
    nodes = B * sum(min(1 << t, total) for t in range(stages))
    xp_rgsw = B * (d1.bit_length() - 1) * ell
    xp_col = B * (d1 - 1)

    def fma_ms(units, transforms, macs):
        cyc = units * (transforms * bfly * 8 + macs * 4) / 32
        return cyc / (sms * 4 * clk_hz) * 1e3

    eq_tr, eq_mac = k + k * (ell - 1), 2 * k * ell * n
    xp_tr, xp_mac = 2 * k + 2 * k * (ell - 1), 4 * k * ell * n
    out = {}
    for name, units, tr, mac in (("ExpandQuery", nodes, eq_tr, eq_mac), ("RgswAssembly", xp_rgsw, xp_tr, xp_mac),
                                 ("ColTor", xp_col, xp_tr, xp_mac)):
        floor = fma_ms(units, tr, mac)
        out[name] = {"bound": "FMA-heavy pipe (IMAD / IMAD.HI)", "floor_ms": floor,
                     "measured_ms": phases[name], "frac": floor / phases[name] if phases[name] else None}
    floor = rs_bytes / (hbm_gbs * 1e9) * 1e3
    out["RowSel"] = {"bound": "HBM", "floor_ms": floor, "measured_ms": phases["RowSel"],
                     "frac": floor / phases["RowSel"] if phases["RowSel"] else None}
    return out


def synthetic_material(G, params, B, stages, rng):
    """Uniform-random key and query material (all kernels are data-oblivious)."""
    b = params.basis
    k, n, ell = b.k, b.n, params.gadget.ell
    qs = np.array([m.q for m in b.moduli], dtype=np.uint64)[:, None]

    def uni(*shape):
        return (rng.integers(0, 1 << 62, size=shape + (k, n), dtype=np.uint64) % qs).astype(np.uint32)

    evks = uni(B, stages, ell, 2)
    rgsw = uni(B, 2 * ell, 2)
    queries = uni(B, 2)
    return evks, rgsw, queries


def cpu_reference(cfg_id, steps, warmup_cap=1):
    """Time the CPU oracle port of answer_batch on a bounded sample: one query
    at the workload's geometry per step.  Returns (qps, seconds, cores, sample)."""
    import numba

    from oracle import gpir_oracle as O

    d0, d1, B, rb, pb, _ = CONFIGS[cfg_id]
    cores = os.cpu_count() or 1
    numba.set_num_threads(cores)
    po = O.default_params(plain_bits=pb)
    R = po.ring
    rng = np.random.default_rng(1)
    total = O.expansion_leaves(d0, d1, po.ell)
    st = O.expand_stages(total)
    uni = lambda *s: np.stack([rng.integers(0, q, size=s + (R.n,), dtype=np.uint64) for q in R.qs], axis=-2)
    db = uni(d1, d0).reshape(d1, d0, R.k * R.n)
    evk, rg = uni(1, st, po.ell, 2), uni(1, 2 * po.ell, 2)
    # warm the numba transforms (JIT compile) on a tiny call
    O.ntt(uni(2), R)
    O.intt(uni(2), R)
    times = []
    for s in range(steps):
        q = uni(1, 2)
        t0 = time.perf_counter()
        O.answer_batch(q, evk, rg, db, d0, d1, po)
        times.append(time.perf_counter() - t0)
    sec = float(np.mean(times))
    return 1.0 / sec, sec, cores, f"1 query/step at {d0}x{d1} (P=2^{pb}) geometry, random key/query material, " \
                                  f"numba NTT on {cores} threads, numpy elsewhere"


def run_reference(args, rank, world):
    if rank != 0:
        return
    d0, d1, B, rb, pb, desc = config_of(args)
    qps, sec, cores, sample = cpu_reference(args.config, args.steps)
    tr = ncu_traffic() if args.config == 2 else None  # the committed capture is of the config-2 launch
    line = {
        "metric": "PIR queries/sec (batched)", "value": qps, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32 (mod-q int64 products)", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": desc, "d0": d0, "d1": d1, "global_batch": B, "record_bytes": rb, "plain_bits": pb},
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import ctypes as C

    import torch

    import paper_2604_04696_b200 as G
    from paper_2604_04696_b200 import _native as nat

    torch.cuda.set_device(local_rank)
    dev = local_rank
    d0, d1, B, rb, pb, desc = config_of(args)
    params = G.HeParams(G.default_basis(4096), pb)
    cfg = G.DbConfig(d0, d1, rb)
    rng = np.random.default_rng(1000 + rank)
    recs = rng.integers(0, 256, size=(cfg.records, rb), dtype=np.uint8)
    db = G.encode_database_array(recs, cfg, params, device=dev)
    del recs
    ctx = db.ctx
    lib = ctx.lib
    total = G.planner.expansion_leaves(d0, d1, params.gadget.ell)
    stages = G.planner.num_expand_stages(total)
    if args.material == "gpu":  # B distinct real clients: keys and queries generated on the GPU
        from paper_2604_04696_b200 import client

        coords = [(int(rng.integers(0, d0)), int(rng.integers(0, d1))) for _ in range(B)]
        if args.clients == "single":  # one client's B queries (the reference's run_bench, src/server.py:416-417)
            sk = client.keygen(ctx, params, 0, d0, d1, seed=7000)
            queries = client.queries(ctx, params, sk, d0, d1, coords, seed=9000)
        else:
            queries = np.concatenate([client.queries(ctx, params, client.keygen(ctx, params, b, d0, d1, seed=7000 + b),
                                                     d0, d1, [coords[b]], seed=9000 + b) for b in range(B)])
    else:
        evks, rgsw, queries = synthetic_material(G, params, B, stages, rng)
        for b in range(B):
            nat.check(lib.gpir_keys_put(ctx.h, b, nat.ptr(np.ascontiguousarray(evks[b])), stages,
                                        nat.ptr(np.ascontiguousarray(rgsw[b]))), "keys")
    slots = np.zeros(B, dtype=np.int32) if args.clients == "single" else np.arange(B, dtype=np.int32)
    words = queries.size
    d_q = torch.from_numpy(queries.view(np.int32).reshape(-1)).to(f"cuda:{dev}")
    d_o = torch.empty_like(d_q)
    # a dedicated stream: the legacy default stream (handle 0) cannot be graph-captured
    stream = torch.cuda.Stream(dev)
    sptr = C.c_void_p(stream.cuda_stream)
    em = np.zeros(16, np.uint8)
    cm = np.zeros(16, np.uint8)
    nat.check(lib.gpir_plan(ctx.h, d0, d1, B, nat.ptr(em, C.c_uint8), 16, nat.ptr(cm, C.c_uint8), 16), "plan")
    if args.modes in ("fused", "op"):
        em[:] = 1 if args.modes == "fused" else 0
        cm[:] = em[0]
    elif args.modes:  # explicit per-stage plan "EQ/CT", chars o (op-level), F (fused), S (split), H (op iNTT+Dcp, fused NTT+MAC)
        code = {"o": 0, "F": 1, "S": 2, "H": 3}
        eq, ct = args.modes.split("/")
        for i, ch in enumerate(eq):
            em[i] = code[ch]
        for i, ch in enumerate(ct):
            cm[i] = code[ch]
    st = nat.GpirStats()

    def step(stats=None):
        nat.check(lib.gpir_answer_batch_dev(ctx.h, db.handle, C.c_void_p(d_q.data_ptr()),
                                            nat.ptr(slots, C.c_int32), B, nat.ptr(em, C.c_uint8), 16,
                                            nat.ptr(cm, C.c_uint8), 16, C.c_void_p(d_o.data_ptr()), sptr,
                                            C.byref(stats) if stats is not None else None), "answer")

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # phase breakdown + RowSel kernel duration, CUDA events on the launch stream (untimed pass)
    ph = {"ExpandQuery": [], "RgswAssembly": [], "RowSelPack": [], "RowSel": [], "ColTor": [], "total": []}
    launches = 0
    for _ in range(max(1, min(args.steps, 5))):
        step(st)
        ph["ExpandQuery"].append(st.ms_expand)
        ph["RgswAssembly"].append(st.ms_rgsw)
        ph["RowSelPack"].append(st.ms_rowsel - st.ms_rowsel_kernel)
        ph["RowSel"].append(st.ms_rowsel_kernel)
        ph["ColTor"].append(st.ms_coltor)
        ph["total"].append(st.ms_total)
        launches = st.launches + 2
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        torch.distributed.barrier()
    qps = world * B / (ms / 1e3)

    # e2e: the C-ABI host entry point with pinned host buffers
    h_q = torch.from_numpy(queries.view(np.int32).reshape(-1)).pin_memory()
    h_o = torch.empty_like(h_q).pin_memory()

    def e2e_step():
        nat.check(lib.gpir_answer_batch(ctx.h, db.handle, C.cast(h_q.data_ptr(), nat._u32p),
                                        nat.ptr(slots, C.c_int32), B, nat.ptr(em, C.c_uint8), 16,
                                        nat.ptr(cm, C.c_uint8), 16, C.cast(h_o.data_ptr(), nat._u32p), None),
                  "answer(host)")

    for _ in range(2):
        e2e_step()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    e2e_s = (time.perf_counter() - t0) / args.steps
    if world > 1:
        t = torch.tensor([e2e_s], device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_qps = world * B / e2e_s

    if rank != 0:
        return
    hbm, peak_kind = _peaks()
    KN = params.basis.k * params.basis.n
    rs_bytes = d0 * d1 * KN * 4 + B * d0 * 2 * KN * 4 + B * d1 * 2 * KN * 4
    rs_ms = float(np.mean(ph["RowSel"]))
    achieved = rs_bytes / (rs_ms / 1e3) / 1e9
    tr = ncu_traffic() if args.config == 2 else None  # the committed capture is of the config-2 launch
    line = {
        "metric": "PIR queries/sec (batched)", "value": qps, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32 (mod-q, 64-bit lazy products)",
        "data": (f"synthetic random records; {'B distinct clients' if args.clients == 'distinct' else 'one client'}"
                 "'s keys and queries generated on the GPU (paper_2604_04696_b200.client)".replace("clients's", "clients'")
                 if args.material == "gpu" else
                 "synthetic (random records, uniform-random key/query material)"),
        "config": {"workload": desc, "d0": d0, "d1": d1, "global_batch": B * world, "per_gpu_batch": B,
                   "record_bytes": rb, "plain_bits": pb, "encoded_db_bytes": d0 * d1 * KN * 4,
                   "l2": f"inputs larger than L2 ({d0 * d1 * KN * 4 >> 30} GiB DB streamed by RowSel every step)",
                   "cuda_graph": "timed steps replay the pipeline as a CUDA graph (library default, recorded during "
                                 "warm-up); phases_ms come from eager passes with per-phase events",
                   "clients": f"{B} distinct" if args.clients == "distinct" else "1 (all B queries from one client)",
                   "parallelism": "replica" if world > 1 else "single",
                   "plan_eq": "".join("oFSH"[v] for v in em[:stages]),
                   "plan_ct": "".join("oFSH"[v] for v in cm[:max(d1.bit_length() - 1, 0)]),
                   "plan_legend": "per stage: o operation-level, H stage-level (digit NTT + key-switch MAC fused), "
                                  "F node-fused, S split"},
        "phases_ms": {k: float(np.mean(v)) for k, v in ph.items()},
        "phase_roofline": phase_rooflines(d0, d1, B, params.basis.k, params.basis.n, params.gadget.ell,
                                          {k: float(np.mean(v)) for k, v in ph.items()}, rs_bytes, hbm),
        "gpu_launches": launches * args.steps,
        "e2e": {"value": e2e_qps, "unit": "queries/s", "h2d_bytes_per_step": words * 4,
                "d2h_bytes_per_step": words * 4},
        "roofline": {"kernel": f"k_rowsel_tc (RowSel, tcgen05.mma kind::i8, M={min(2 * B, 128)} tiles)", "bound": "hbm",
                     "achieved": achieved, "peak": hbm,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": tr[0] if tr else None,
                     "traffic_src": f"profiles/{tr[1]} ({tr[2]}, ncu --set full)" if tr else None,
                     "algorithmic_bytes": rs_bytes, "avg_launch_ms": rs_ms},
        "dominant_kernel": dominant_kernel(),
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu:
        cq, csec, cores, sample = cpu_reference(args.config, 1)
        line["cpu_baseline"] = {"value": cq, "unit": "queries/s", "cores": cores, "kind": "port", "sample": sample}
    print(json.dumps(line), flush=True)


def run_sharded(args, rank, world, local_rank):
    """Multi-GPU sharded serving (paper_2604_04696_b200/cluster.py), strong
    scaling: the config's DB and batch are fixed and split over the ranks.
    rowshard: DB rows + query owners, NCCL all-to-all + reduce-scatter(sum)
    (the north star's modular-add combine).  colshard: DB columns + query owners,
    NCCL all-gather of the row cts + all-to-all of one partial per query (the
    reference's SHARD_ALL_GATHER)."""
    import torch
    import torch.distributed as dist

    import paper_2604_04696_b200 as G
    from paper_2604_04696_b200.cluster import (CudaColShard, CudaRowShard, TorchComm, answer_col_sharded,
                                               answer_row_sharded)

    torch.cuda.set_device(local_rank)
    d0, d1, B, rb, pb, desc = config_of(args)
    col = args.strategy == "colshard"
    if B % world or (d1 if col else d0) % world:
        raise SystemExit(f"batch {B} / {'d1' if col else 'd0'} do not split over {world} ranks")
    params = G.HeParams(G.default_basis(4096), pb)
    b_own = B // world
    rng = np.random.default_rng(500 + rank)
    if col:
        recs = rng.integers(0, 256, size=(d0 * (d1 // world), rb), dtype=np.uint8)
        be = CudaColShard(params, recs, d0, d1, rb, world, local_rank)
    else:
        recs = rng.integers(0, 256, size=((d0 // world) * d1, rb), dtype=np.uint8)
        be = CudaRowShard(params, recs, d0, d1, rb, world, local_rank)
    del recs
    stages = G.planner.num_expand_stages(G.planner.expansion_leaves(d0, d1, params.gadget.ell))
    evks, rgsw, queries = synthetic_material(G, params, b_own, stages, rng)
    for b in range(b_own):
        be.put_keys(b, evks[b], rgsw[b])
    slots = np.arange(b_own, dtype=np.int32)
    q = torch.from_numpy(queries.view(np.int32)).cuda()

    class _One:  # world 1: the collectives are identities
        size = 1
        all_to_all = staticmethod(lambda x: x)
        reduce_scatter_sum = staticmethod(lambda x: x[0])
        all_gather = staticmethod(lambda x: x.unsqueeze(0))

    comm = TorchComm() if world > 1 else _One()
    answer = answer_col_sharded if col else answer_row_sharded
    step = lambda: answer(be, comm, q, slots, d0, d1)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if rank == 0:
        par = (f"colshard{world} (DB columns + query owners; NCCL all-gather + all-to-all)" if col else
               f"rowshard{world} (DB rows + query owners; NCCL all-to-all + reduce-scatter)")
        line = {
            "metric": "PIR queries/sec (batched)", "value": B / (ms / 1e3), "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32 (mod-q, 64-bit lazy products)",
            "data": "synthetic (random records, uniform-random key/query material)",
            "config": {"workload": desc, "d0": d0, "d1": d1, "global_batch": B, "record_bytes": rb, "plain_bits": pb,
                       "parallelism": par},
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--modes", default="", help='"fused", "op", or an explicit plan "EQ/CT" (o/F/S/H per stage)')
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--material", default="gpu", choices=["gpu", "uniform"],
                    help="client keys/queries: real ones generated on the GPU, or uniform-random residues")
    ap.add_argument("--batch", type=int, default=0, help="override the config's batch size (batch sweeps)")
    ap.add_argument("--clients", default="distinct", choices=["distinct", "single"],
                    help="B distinct clients (worst-case key traffic, default) or one client's B queries")
    ap.add_argument("--strategy", default="replica", choices=["replica", "rowshard", "colshard"],
                    help="multi-GPU mode: replica (DB copy + own batch per GPU), rowshard (north-star DB row "
                         "shards, modular-add combine) or colshard (DB column shards, all-gather)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        if args.impl == "ours":
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
        else:
            dist.init_process_group("gloo")
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif args.strategy in ("rowshard", "colshard"):
        run_sharded(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
