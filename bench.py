"""GPIR server-pipeline benchmark (BASELINE.json metric: PIR queries/sec, batched).

One step = one full batch through the server pipeline (ExpandQuery -> RGSW
assembly -> RowSel -> ColTor) for B client queries against the encoded DB.
Default workload = BASELINE configs[2], the largest single-GPU configuration:
8 GiB encoded DB (D0=256 x D1=512 polys, 8 KiB records at P=2^16), a batch of
128 distinct clients, one B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config 1..5] [--strategy auto|rowshard|colshard|replica]

`value` is device-timed QPS with queries resident in HBM (CUDA events on the
launch stream); `e2e` is the same metric through the C ABI host entry point
`gpir_answer_batch` with pinned host buffers (H2D of queries + D2H of
responses inside the timed region).  `--impl reference` times the reference's
own CPU implementation (latpir, installed in baseline/_ref; the oracle port if
it is absent) on this host: a bounded sample per step, extrapolated to the
config (see RefSampler).  `--gpus N` without a torchrun environment re-launches
itself under torch.distributed.run with N ranks (one per GPU).  N > 1 shards
the DB: by rows (the north star; configs 1-3) or by columns (configs 4-5,
whose DBs do not fit one GPU), see paper_2604_04696_b200/cluster.py.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(ROOT, ".numba_cache"))

CONFIGS = {
    # id: (d0, d1 per GPU, B, record_bytes, plain_bits, description)
    1: (16, 16, 1, 16384, 32, "config1: 16 MiB encoded DB (16x16, 16 KiB records, P=2^32), 1 query"),
    2: (256, 64, 32, 8192, 16, "config2: 1 GiB encoded DB (256x64 polys, 8 KiB records, P=2^16), batch 32 clients"),
    3: (256, 512, 128, 8192, 16, "config3: 8 GiB encoded DB (256x512 polys, 8 KiB records, P=2^16), batch 128 clients"),
    4: (256, 2048, 256, 8192, 16, "config4: 32 GiB encoded DB (256x2048 polys, 8 KiB records, P=2^16), batch 256 clients"),
    5: (256, 4096, 512, 8192, 16, "config5: capacity, 64 GiB encoded DB per GPU (256 x 4096N polys on N GPUs: "
                                  "512 GiB at N=8, 8 KiB records, P=2^16), batch 512 clients"),
}
DEFAULT_CONFIG = 3
INT8_TOPS_PEAK = 4769.0  # tcgen05.mma kind::i8 M128xN32xK32 every 16.0 cycles per SM (profiles/r1f_umma.txt) x 148 x 1.965 GHz


def config_of(args, world=1):
    """(d0, d1, B, record_bytes, plain_bits, description) of the run; config 5's DB grows with the ranks,
    --batch overrides the batch (a sweep at the same DB geometry)."""
    d0, d1, B, rb, pb, desc = CONFIGS[args.config]
    if args.config == 5:
        d1 *= world
    if getattr(args, "batch", 0):
        desc = f"{desc.split(', batch')[0]}, batch {args.batch} (sweep; the config's own batch is {B})"
        B = args.batch
    return d0, d1, B, rb, pb, desc


def strategy_of(args, world):
    if world == 1:  # an explicit sharded strategy on one GPU runs its orchestration with identity collectives
        return args.strategy if args.strategy in ("rowshard", "colshard") else "single"
    if args.strategy != "auto":
        return args.strategy
    B = config_of(args, world)[2]
    if B % world:  # a batch that does not split over the ranks (config 1: B = 1): one copy per GPU
        return "replica"
    return "colshard" if args.config >= 4 else "rowshard"


def parallelism_of(strategy, world):
    return {"single": "single",
            "replica": f"replica{world} (own DB copy + own batch per GPU)",
            "rowshard": f"rowshard{world} (DB rows + query owners; NCCL all-to-all + reduce-scatter modular add)",
            "colshard": f"colshard{world} (DB columns + query owners; NCCL all-gather + all-to-all)"}[strategy]


def common_config(args, world):
    """The workload description both arms print (the driver compares the arms' configs)."""
    d0, d1, B, rb, pb, desc = config_of(args, world)
    strat = strategy_of(args, world)
    gb = B * world if strat == "replica" else B
    kn = 4096 * 4
    return {"workload": desc, "d0": d0, "d1": d1, "global_batch": gb, "record_bytes": rb, "plain_bits": pb,
            "encoded_db_bytes": d0 * d1 * kn * 4, "parallelism": parallelism_of(strat, world),
            "l2": f"inputs larger than L2 (the {d0 * d1 * kn * 4 / 2**30:g} GiB DB is streamed by RowSel every step)"
            if d0 * d1 * kn * 4 > 126 * 2**20 else "DB fits L2 (config 1: the SPEC toy case)"}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


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


# ---------------------------------------------------------------------------
# committed ncu evidence (profiles/*_c<config>_ncu.json, tools/ncu_summary.py)

def _profile(cfg_id):
    """The newest committed ncu summary of this config's bench step (launch list + full captures)."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"*_c{cfg_id}_ncu.json")), key=os.path.getmtime)
    for f in reversed(files):
        try:
            return json.load(open(f)), os.path.basename(f)
        except Exception:
            continue
    return None, None


def ncu_traffic(cfg_id, prefix):
    """DRAM read + write bytes of the kernel over one bench step of this config: the sum over
    its launches in the committed ncu launch list (several launches when the capacity path runs
    RowSel per column window), else the full capture of its first launch."""
    js, name = _profile(cfg_id)
    if not js:
        return None
    for k, d in (js.get("launch_list") or {}).items():
        if k.startswith(prefix):
            return d["dram_read"] + d["dram_write"], name, f"{k}, {d['launches']} launch(es), launch list"
    for k, d in js.get("kernels", {}).items():
        if k.startswith(prefix) and "traffic_bytes" in d:
            return d["traffic_bytes"], name, f"{k}, --set full"
    return None


def dominant_kernel(cfg_id):
    """Largest-share kernel of this config's committed ncu launch list, with its pipe
    counters when a full capture of it is committed."""
    js, name = _profile(cfg_id)
    if not js or not js.get("launch_list"):
        return None
    ll = js["launch_list"]
    tot = sum(v["ns"] for v in ll.values())
    kname, v = max(ll.items(), key=lambda kv: kv[1]["ns"])
    full = js.get("kernels", {}).get(kname, {})

    def pct(key):
        m = full.get(key)
        return float(str(m["value"]).replace(",", "")) / 100 if isinstance(m, dict) else None

    return {"kernel": kname, "share_of_launch_list": v["ns"] / tot, "launches": v["launches"],
            "bound": "FMA-heavy integer pipe (IMAD, IMAD.HI/WIDE)",
            "fmaheavy_busy": pct("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "phase_floor_frac": "see phase_roofline (live)",
            "src": f"profiles/{name} (ncu launch list + --set full of config {cfg_id})"}


def phase_rooflines(d0, d1, B, k, n, ell, phases, rs_bytes, hbm_gbs, sms=148, clk_hz=1.965e9):
    """Per-phase roofline fractions.  The tree phases (ExpandQuery, RGSW
    assembly, ColTor) are bound by the FMA-heavy integer pipe: a Shoup
    butterfly is one IMAD.HI (quarter rate) + two IMADs (half rate) = 8
    SMSP-cycles per warp, an exact 64-bit MAC one IMAD.WIDE = 4 (measured,
    tools/micro/pipes.cu).  Algorithmic work per node / external product, with
    the top gadget digit folded into the keys: ExpandQuery node =
    k iNTTs + k (ell-1) digit NTTs, 2 k ell n MACs; external product = 2 k iNTTs
    + 2 k (ell-1) digit NTTs, 4 k ell n MACs.  RowSel (GEMM + output transpose +
    A-operand pack) is bound by the larger of its HBM and int8 tensor floors."""
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
    ops = 2 * 16 * k * n * 2 * B * d0 * d1  # byte-plane MACs, 2 ops each
    floor = max(rs_bytes / (hbm_gbs * 1e9), ops / (INT8_TOPS_PEAK * 1e12)) * 1e3
    rs = phases["RowSel"] + phases.get("RowSelTranspose", 0.0) + phases.get("RowSelPack", 0.0)
    out["RowSel"] = {"bound": "max(HBM, int8 tensor)", "floor_ms": floor, "measured_ms": rs,
                     "frac": floor / rs if rs else None, "parts": "GEMM + output transpose + A-operand pack"}
    return out


def rowsel_roofline(d0, d1, B, kn, ms, hbm, peak_kind, cfg_id):
    """The RowSel GEMM kernel against its binding roofline: the algorithmic bytes
    (src/planner.py:233-238) at the measured HBM bandwidth, or the byte-plane MACs at
    the int8 tensor-core peak, whichever floor is larger."""
    rs_bytes = d0 * d1 * kn * 4 + B * d0 * 2 * kn * 4 + B * d1 * 2 * kn * 4
    ops = 2 * 16 * kn * 2 * B * d0 * d1
    t_hbm, t_tc = rs_bytes / (hbm * 1e9), ops / (INT8_TOPS_PEAK * 1e12)
    tk = 2 * B > 64 and d0 <= 256
    kname = "k_rowsel_tk" if tk else "k_rowsel_tc"
    tr = ncu_traffic(cfg_id, kname)
    if t_tc > t_hbm:
        r = {"bound": "tensor", "achieved": ops / (ms / 1e3) / 1e12, "peak": INT8_TOPS_PEAK, "unit": "TFLOP/s",
             "peak_kind": "measured instruction rate (tcgen05.mma kind::i8, int8 TOP/s, profiles/r1f_umma.txt)",
             "algorithmic_ops": ops}
    else:
        r = {"bound": "hbm", "achieved": rs_bytes / (ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
             "peak_kind": peak_kind}
    r.update({"kernel": f"{kname} (RowSel GEMM, tcgen05.mma kind::i8 byte planes)", "frac": r["achieved"] / r["peak"],
              "traffic": tr[0] if tr else None,
              "traffic_src": f"profiles/{tr[1]} ({tr[2]})" if tr else None,
              "algorithmic_bytes": rs_bytes, "avg_launch_ms": ms,
              "floors_ms": {"hbm": t_hbm * 1e3, "tensor": t_tc * 1e3}})
    return r


# ---------------------------------------------------------------------------
# the reference's CPU path (bounded sample, extrapolated)

def _latpir():
    p = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(p, "latpir")):
        if p not in sys.path:
            sys.path.insert(0, p)
        try:
            import latpir  # noqa: F401
            return True
        except Exception:
            return False
    return False


class RefSampler:
    """Times the reference's answer_batch on a bounded sample of the workload:
    bs = min(B, 2) queries of bs distinct clients against a d0 x d1s slice of the
    DB (d1s = min(d1, 16) columns; the full config when it is that small), and
    extrapolates each phase to the full geometry in D1 only:
    ExpandQuery x nodes(d1)/nodes(d1s), RGSW assembly x log2 d1 / log2 d1s,
    RowSel x d1 / d1s, ColTor x (d1 - 1)/(d1s - 1).  Per-query cost is taken at
    the sample's batch (the CPU's per-query cost at B=128 would need minutes per
    step).  Runs latpir (baseline/_ref, the unmodified reference, kind
    "reference") when installed, else the oracle port (kind "port")."""

    def __init__(self, cfg_id, world=1, seed=1):
        d0, d1, B, rb, pb, _ = CONFIGS[cfg_id]
        if cfg_id == 5:
            d1 *= world
        self.d0, self.d1, self.B = d0, d1, B
        self.d1s, self.bs = min(d1, 16), min(B, 2)
        self.cores = os.cpu_count() or 1
        os.environ.setdefault("NUMBA_NUM_THREADS", str(self.cores))
        self.kind = "reference" if _latpir() else "port"
        rng = np.random.default_rng(seed)
        if self.kind == "reference":
            from latpir import he, ring
            from latpir.protocol import ClientSession, DbConfig, ServeStats, answer_batch, encode_database

            P = he.default_params() if pb == 32 else he.HeParams(ring.default_basis(4096), pb)
            cfg = DbConfig(d0, self.d1s, rb)
            recs = [rng.integers(0, 256, size=rb, dtype=np.uint8).tobytes() for _ in range(cfg.records)]
            self.db = encode_database(recs, cfg, P)
            sess = [ClientSession.create(P, cfg, rng, client_id=c) for c in range(self.bs)]
            self.keys = {s.client_id: s.keys for s in sess}
            self.queries = [s.gen_query(int(rng.integers(d0)), int(rng.integers(self.d1s)), rng) for s in sess]
            self.P, self._answer, self._stats = P, answer_batch, ServeStats
            self._answer(self.queries[:1], self.keys, self.db, self.P)  # numba JIT warm-up
        else:
            import numba

            from oracle import gpir_oracle as O

            numba.set_num_threads(self.cores)
            po = O.default_params(plain_bits=pb)
            R = po.ring
            total = O.expansion_leaves(d0, self.d1s, po.ell)
            st = O.expand_stages(total)
            uni = lambda *s: np.stack([rng.integers(0, q, size=s + (R.n,), dtype=np.uint64) for q in R.qs], axis=-2)
            self.db = uni(self.d1s, d0).reshape(self.d1s, d0, R.k * R.n)
            self.evk, self.rg, self.q = uni(self.bs, st, po.ell, 2), uni(self.bs, 2 * po.ell, 2), uni(self.bs, 2)
            self.po, self.O = po, O
            O.ntt(uni(2), R)
            O.intt(uni(2), R)

    def sample(self) -> str:
        tag = "latpir.protocol.answer_batch (baseline/_ref)" if self.kind == "reference" else \
            "oracle port of answer_batch (numpy + numba NTT)"
        ex = "" if (self.d1s, self.bs) == (self.d1, self.B) else \
            f"; extrapolated in D1 from a {self.d0}x{self.d1s} slice at B={self.bs} ({self.bs} distinct clients)"
        return f"{tag}, {self.cores} host threads{ex}"

    def step(self):
        """One timed sample; returns (sample seconds, extrapolated seconds per query)."""
        t0 = time.perf_counter()
        if self.kind == "reference":
            st = self._stats()
            self._answer(self.queries, self.keys, self.db, self.P, stats=st)
            ph = dict(st.phase_seconds)
        else:
            ph = {}
            self.O.answer_batch(self.q, self.evk, self.rg, self.db, self.d0, self.d1s, self.po, stats=ph)
        sec = time.perf_counter() - t0
        return sec, self.extrapolate(ph, sec) / self.bs

    def extrapolate(self, ph, sec):
        if (self.d1s, self.bs) == (self.d1, self.B) or not ph:
            return sec
        ell = 5

        def nodes(d1):
            total = self.d0 + (d1.bit_length() - 1) * ell
            return sum(min(1 << t, total) for t in range((total - 1).bit_length()))

        lb = lambda d: max(d.bit_length() - 1, 1)
        f = {"ExpandQuery": nodes(self.d1) / nodes(self.d1s), "RgswAssembly": lb(self.d1) / lb(self.d1s),
             "RowSel": self.d1 / self.d1s, "ColTor": (self.d1 - 1) / max(self.d1s - 1, 1)}
        rest = sec - sum(ph.values())
        return sum(v * f.get(k, 1.0) for k, v in ph.items()) + max(rest, 0.0)


def run_reference(args, rank, world):
    if rank != 0:
        return
    ref = RefSampler(args.config, world)
    for _ in range(min(args.warmup, 1)):  # a warm-up sample (beyond the JIT warm-up in the constructor)
        ref.step()
    samples, per_q = [], []
    for _ in range(args.steps):
        s, q = ref.step()
        samples.append(s)
        per_q.append(q)
    qps = 1.0 / float(np.mean(per_q))
    B = common_config(args, world)["global_batch"]
    line = {
        "metric": "PIR queries/sec (batched)", "value": qps, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": B / qps * 1e3, "higher_is_better": True,
        "scaling": "weak" if args.config == 5 else "strong", "vs_baseline": None,
        "dtype": "u64 (mod-q int64 products, numpy)", "data": "synthetic (random records, reference client keys/queries)",
        "impl": "reference", "config": common_config(args, world),
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": ref.cores, "kind": ref.kind,
                         "sample": ref.sample(), "sample_seconds_per_step": float(np.mean(samples))},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "extrapolated": (ref.d1s, ref.bs) != (ref.d1, ref.B),
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(args, world=1):
    ref = RefSampler(args.config, world)
    sec, per_q = ref.step()
    return {"value": 1.0 / per_q, "unit": "queries/s", "cores": ref.cores, "kind": ref.kind, "sample": ref.sample(),
            "sample_seconds": sec}


# ---------------------------------------------------------------------------
# our arm

def _device_records(torch, n_rec, rb, dev, seed):
    g = torch.Generator(device=f"cuda:{dev}")
    g.manual_seed(seed)
    return torch.randint(0, 256, (n_rec, rb), dtype=torch.uint8, device=f"cuda:{dev}", generator=g)


def _client_material(G, ctx, params, d0, d1, B, rng, args, lib, nat, slot0=0):
    """B distinct clients' keys (into key slots slot0..) and queries, generated on the GPU."""
    stages = G.planner.num_expand_stages(G.planner.expansion_leaves(d0, d1, params.gadget.ell))
    coords = [(int(rng.integers(0, d0)), int(rng.integers(0, d1))) for _ in range(B)]
    if args.material == "gpu":
        from paper_2604_04696_b200 import client

        if args.clients == "single":
            sk = client.keygen(ctx, params, slot0, d0, d1, seed=7000)
            q = client.queries(ctx, params, sk, d0, d1, coords, seed=9000)
            return q, np.full(B, slot0, dtype=np.int32)
        q = np.concatenate([client.queries(ctx, params, client.keygen(ctx, params, slot0 + b, d0, d1, seed=7000 + b),
                                           d0, d1, [coords[b]], seed=9000 + b) for b in range(B)])
        return q, np.arange(slot0, slot0 + B, dtype=np.int32)
    b_ = params.basis
    qs = np.array([m.q for m in b_.moduli], dtype=np.uint64)[:, None]
    uni = lambda *s: (rng.integers(0, 1 << 62, size=s + (b_.k, b_.n), dtype=np.uint64) % qs).astype(np.uint32)
    for b in range(1 if args.clients == "single" else B):
        nat.check(lib.gpir_keys_put(ctx.h, slot0 + b, nat.ptr(np.ascontiguousarray(uni(stages, params.gadget.ell, 2))),
                                    stages, nat.ptr(np.ascontiguousarray(uni(2 * params.gadget.ell, 2)))), "keys")
    slots = np.full(B, slot0, dtype=np.int32) if args.clients == "single" else np.arange(slot0, slot0 + B,
                                                                                         dtype=np.int32)
    return uni(B, 2), slots


def run_ours(args, rank, world, local_rank):
    """One GPU per rank serving the whole config (world 1) or its own batch against its own DB copy (replica)."""
    import ctypes as C

    import torch

    import paper_2604_04696_b200 as G
    from paper_2604_04696_b200 import _native as nat

    torch.cuda.set_device(local_rank)
    dev = local_rank
    d0, d1, B, rb, pb, desc = config_of(args, 1)
    params = G.HeParams(G.default_basis(4096), pb)
    cfg = G.DbConfig(d0, d1, rb)
    rng = np.random.default_rng(1000 + rank)
    compact = args.config >= 4  # capacity configs: only the byte-plane image stays resident
    recs = _device_records(torch, cfg.records, rb, dev, 1000 + rank)
    db = G.encode_database_device(recs, cfg, params, compact=compact)
    del recs
    torch.cuda.empty_cache()
    ctx = db.ctx
    lib = ctx.lib
    stages = G.planner.num_expand_stages(G.planner.expansion_leaves(d0, d1, params.gadget.ell))
    queries, slots = _client_material(G, ctx, params, d0, d1, B, rng, args, lib, nat)
    words = queries.size
    d_q = torch.from_numpy(queries.view(np.int32).reshape(-1)).to(f"cuda:{dev}")
    d_o = torch.empty_like(d_q)
    stream = torch.cuda.Stream(dev)  # the legacy default stream (handle 0) cannot be graph-captured
    sptr = C.c_void_p(stream.cuda_stream)
    em = np.zeros(16, np.uint8)
    cm = np.zeros(16, np.uint8)
    nat.check(lib.gpir_plan(ctx.h, d0, d1, B, nat.ptr(em, C.c_uint8), 16, nat.ptr(cm, C.c_uint8), 16), "plan")
    if args.modes in ("fused", "op"):
        em[:] = 1 if args.modes == "fused" else 0
        cm[:] = em[0]
    elif args.modes:  # explicit per-stage plan "EQ/CT", chars o (op-level), F (fused), S (split), H (stage-level)
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
    # phase breakdown + RowSel kernel durations, CUDA events on the launch stream (untimed passes)
    ph = {k: [] for k in ("ExpandQuery", "RgswAssembly", "RowSelPack", "RowSel", "RowSelTranspose", "ColTor",
                          "total")}
    launches = 0
    for _ in range(max(1, min(args.steps, 3))):
        step(st)
        ph["ExpandQuery"].append(st.ms_expand)
        ph["RgswAssembly"].append(st.ms_rgsw)
        ph["RowSelPack"].append(max(st.ms_rowsel - st.ms_rowsel_kernel - st.ms_rowsel_transpose, 0.0))
        ph["RowSel"].append(st.ms_rowsel_kernel)
        ph["RowSelTranspose"].append(st.ms_rowsel_transpose)
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
    phases = {k: float(np.mean(v)) for k, v in ph.items()}
    rs_bytes = d0 * d1 * KN * 4 + B * d0 * 2 * KN * 4 + B * d1 * 2 * KN * 4
    line = {
        "metric": "PIR queries/sec (batched)", "value": qps, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak" if world > 1 else "strong", "vs_baseline": None,
        "dtype": "u32 (mod-q residues; int8 tensor-core byte planes, 64-bit lazy products)",
        "data": (f"synthetic: random records generated on the GPU; {'B distinct clients' if args.clients == 'distinct' else 'one client'}"
                 "' keys and queries generated on the GPU (paper_2604_04696_b200.client)"
                 if args.material == "gpu" else "synthetic: random records, uniform-random key/query material"),
        "config": common_config(args, world),
        "run": {"per_gpu_batch": B, "clients": f"{B} distinct" if args.clients == "distinct" else "1",
                "compact_db": compact, "device_db_bytes": db.device_bytes,
                "cuda_graph": "timed steps replay the pipeline as a CUDA graph (library default, recorded during "
                              "warm-up); phases_ms come from eager passes with per-phase events",
                "plan_eq": "".join("oFSH"[v] for v in em[:stages]),
                "plan_ct": "".join("oFSH"[v] for v in cm[:max(d1.bit_length() - 1, 0)]),
                "plan_legend": "per stage: o operation-level, H stage-level (digit NTT + key-switch MAC fused), "
                               "F node-fused, S split"},
        "phases_ms": phases,
        "phase_roofline": phase_rooflines(d0, d1, B, params.basis.k, params.basis.n, params.gadget.ell, phases,
                                          rs_bytes, hbm),
        "gpu_launches": launches * args.steps,
        "e2e": {"value": e2e_qps, "unit": "queries/s", "h2d_bytes_per_step": words * 4,
                "d2h_bytes_per_step": words * 4},
        "roofline": rowsel_roofline(d0, d1, B, KN, phases["RowSel"], hbm, peak_kind, args.config),
        "dominant_kernel": dominant_kernel(args.config),
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args)
    print(json.dumps(line), flush=True)


def run_sharded(args, rank, world, local_rank):
    """Multi-GPU sharded serving (paper_2604_04696_b200/cluster.py): the config's
    DB and batch split over the ranks (config 5: 64 GiB of DB per rank).
    rowshard: DB rows + query owners, NCCL all-to-all + reduce-scatter(sum)
    (the north star's modular-add combine).  colshard: DB columns + query owners,
    NCCL all-gather of the row cts + all-to-all of one partial per query (the
    reference's SHARD_ALL_GATHER)."""
    import torch
    import torch.distributed as dist

    import paper_2604_04696_b200 as G
    from paper_2604_04696_b200.cluster import (CountingComm, CudaColShard, CudaRowShard, Strategy, TorchComm,
                                               answer_col_sharded, answer_row_sharded, device_comm_bytes)

    torch.cuda.set_device(local_rank)
    dev = local_rank
    d0, d1, B, rb, pb, desc = config_of(args, world)
    strat = strategy_of(args, world)
    col = strat == "colshard"
    if B % world or (d1 if col else d0) % world:
        raise SystemExit(f"batch {B} / {'d1' if col else 'd0'} do not split over {world} ranks")
    params = G.HeParams(G.default_basis(4096), pb)
    b_own = B // world
    rng = np.random.default_rng(500 + rank)
    compact = args.config >= 4
    if col:
        recs = _device_records(torch, d0 * (d1 // world), rb, dev, 500 + rank)
        be = CudaColShard(params, recs, d0, d1, rb, world, dev, compact=compact)
    else:
        recs = _device_records(torch, (d0 // world) * d1, rb, dev, 500 + rank)
        be = CudaRowShard(params, recs, d0, d1, rb, world, dev, compact=compact)
    del recs
    torch.cuda.empty_cache()
    from paper_2604_04696_b200 import _native as nat
    queries, slots = _client_material(G, be.ctx, params, d0, d1, b_own, rng, args, be.ctx.lib, nat)
    q = torch.from_numpy(queries.view(np.int32)).to(f"cuda:{dev}")

    class _One:  # world 1: the collectives are identities
        size = 1
        rank = 0
        all_to_all = staticmethod(lambda x: x)
        reduce_scatter_sum = staticmethod(lambda x: x[0])
        all_gather = staticmethod(lambda x: x.unsqueeze(0))

    comm = TorchComm() if world > 1 else _One()
    answer = answer_col_sharded if col else answer_row_sharded
    step = lambda qq, c=comm: answer(be, c, qq, slots, d0, d1)
    for _ in range(args.warmup):
        step(q)
    # one counted batch: the measured exchange volume next to the closed form
    cc = CountingComm(comm)
    step(q, cc)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = int(nat.load().gpir_launch_count())
    with ClockSampler(dev) as clk:
        e0.record()
        for _ in range(args.steps):
            step(q)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    launches = int(nat.load().gpir_launch_count()) - n0  # this rank's libgpir kernels (no graphs here)
    # e2e: this rank's queries from pinned host memory, responses back to the host
    h_q = torch.from_numpy(queries.view(np.int32)).pin_memory()
    h_o = torch.empty((b_own, queries.shape[1] * queries.shape[2] * queries.shape[3]), dtype=torch.int32).pin_memory()

    def e2e_step():
        out = step(h_q.to(f"cuda:{dev}", non_blocking=True))
        h_o.copy_(out.reshape(h_o.shape), non_blocking=True)
        torch.cuda.synchronize()

    e2e_step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    e2e_s = (time.perf_counter() - t0) / args.steps
    stats = torch.tensor([ms, e2e_s, float(cc.ledger.after_expand_bytes), float(cc.ledger.after_coltor_bytes),
                          float(cc.ledger.rgsw_sidecar_bytes)], dtype=torch.float64, device=f"cuda:{dev}")
    if world > 1:
        mx = stats[:2].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = stats[2:].clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        stats = torch.cat([mx, sm])
        clocks = [None] * world
        dist.all_gather_object(clocks, clk.summary())
    else:
        clocks = [clk.summary()]
    ms, e2e_s = float(stats[0]), float(stats[1])
    if rank == 0:
        st = Strategy.SHARD_ALL_GATHER if col else Strategy.ROW_SHARD
        model = device_comm_bytes(st, G.DbConfig(d0, d1, rb), B, world, params)
        line = {
            "metric": "PIR queries/sec (batched)", "value": B / (ms / 1e3), "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak" if args.config == 5 else "strong", "vs_baseline": None,
            "dtype": "u32 (mod-q residues; int8 tensor-core byte planes, 64-bit lazy products)",
            "data": "synthetic: random records generated on the GPU; "
                    + ("B distinct clients' keys and queries generated on the GPU" if args.material == "gpu"
                       else "uniform-random key/query material"),
            "config": common_config(args, world),
            "run": {"per_gpu_batch_owned": b_own, "compact_db": compact},
            "gpu_launches": launches,
            "e2e": {"value": B / e2e_s, "unit": "queries/s", "h2d_bytes_per_step": queries.nbytes * world,
                    "d2h_bytes_per_step": queries.nbytes * world},
            "comm_bytes_per_step": {"measured": {"after_expand": float(stats[2]), "after_coltor": float(stats[3]),
                                                 "rgsw_sidecar": float(stats[4])},
                                    "model": {"after_expand": model.after_expand_bytes,
                                              "after_coltor": model.after_coltor_bytes,
                                              "rgsw_sidecar": model.rgsw_sidecar_bytes}},
            "clocks": clocks[0], "clocks_per_rank": clocks,
        }
        print(json.dumps(line), flush=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--modes", default="", help='"fused", "op", or an explicit plan "EQ/CT" (o/F/S/H per stage)')
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample of the reference")
    ap.add_argument("--material", default="gpu", choices=["gpu", "uniform"],
                    help="client keys/queries: real ones generated on the GPU, or uniform-random residues")
    ap.add_argument("--batch", type=int, default=0, help="override the config's batch size (batch sweeps)")
    ap.add_argument("--clients", default="distinct", choices=["distinct", "single"],
                    help="B distinct clients (worst-case key traffic, default) or one client's B queries")
    ap.add_argument("--strategy", default="auto", choices=["auto", "replica", "rowshard", "colshard"],
                    help="N > 1: auto = rowshard (north-star DB row shards, modular-add combine) for configs 1-3, "
                         "colshard (DB column shards, all-gather) for the capacity configs 4-5")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)]
        os.execv(sys.executable, cmd + sys.argv[1:])
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.impl == "ours":
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    if args.impl == "reference":
        run_reference(args, rank, world)  # rank 0 alone; the others exit without work
    elif strategy_of(args, world) in ("rowshard", "colshard"):
        run_sharded(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)
    if world > 1 and args.impl == "ours":
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
