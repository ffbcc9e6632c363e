"""Benchmark: BFS + cover-edge triangle count on a seeded synthetic graph.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config rmat24]
    python bench.py --impl reference ...      # the CPU reference arm

One step = one pass of the hot path over the device-resident graph: min-id
component roots + multi-source BFS levels -> cover-edge selection ->
per-cover-edge intersection -> exact 64-bit count (tcb_cetc).  Graph
construction is outside the timed region, as in the reference's protocol
(bench.py:1-9 of the reference).  metric = m / t_step (undirected edges/s).

For N > 1 (one rank per GPU, NCCL): every rank holds a replica of the CSR,
labels it, and intersects its 1/N slice of the cover set; the partial
tallies are summed with one all-reduce.  Total work is
fixed as N grows: "scaling": "strong".  `--gpus N` without torchrun starts the
N ranks itself (torch.distributed.run on 127.0.0.1); under torchrun the world
size must equal N.

--impl reference: the reference's CPU path (the oracle's C port of
bfs_levels_k + cetc_sm_range_k, all host threads) over the SAME workload.
The timed region is one complete run, measured, not extrapolated: the
1-core BFS, then CETC-SM over every edge, cut into K contiguous edge ranges
(step k = range k; the K ranges cover every edge exactly once, and their
summed tallies must reproduce T).

Timing: W untimed warm-up steps, then K steps bracketed by barrier +
cuda.synchronize, CUDA events on the launching stream, max over ranks.  The
RMAT-24 CSR (4.3 GB) is larger than the 126 MB L2, so no flush is needed;
smaller configs flush L2 between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "edges/s for BFS + cover-edge triangle count; achieved HBM GB/s vs peak"
UNIT = "edges/s"
L2_BYTES = 126 * 2**20


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="rmat24")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-baseline", default="auto", choices=["auto", "off"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="target CPU seconds for the cpu_baseline sample")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# peaks, clocks


def hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.idx = device_index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
# CPU baseline (oracle = C restatement of the reference; the reference itself
# is pure Python/numba and is not installed on the GPU box)


def cpu_sample(n, row, nb, eu, ev, target_s: float, threads: int):
    """Time the oracle on a bounded sample of the workload: the full
    single-threaded BFS (_kernels.py:129-157) plus CETC-SM
    (_kernels.py:729-755, all threads) over every s-th edge; the full-graph
    time is t_bfs + s * t_sample.  Returns a dict for "cpu_baseline"."""
    import oracle
    m = len(eu)
    t0 = time.perf_counter()
    level, _, _, _ = oracle.bfs_levels(row, nb, n)
    t_bfs = time.perf_counter() - t0
    # probe ~50k evenly spaced edges, then size the sample to ~target_s
    stride = max(1, m // 50_000)
    t0 = time.perf_counter()
    oracle.cetc_sm_counts(row, nb, level, np.ascontiguousarray(eu[::stride]),
                          np.ascontiguousarray(ev[::stride]), threads=threads)
    per_edge = max(time.perf_counter() - t0, 1e-6) / max(1, len(eu[::stride]))
    budget = max(1.0, target_s - t_bfs)
    stride = max(1, int(np.ceil(m * per_edge / budget)))
    sub_u = np.ascontiguousarray(eu[::stride])
    sub_v = np.ascontiguousarray(ev[::stride])
    t0 = time.perf_counter()
    oracle.cetc_sm_counts(row, nb, level, sub_u, sub_v, threads=threads)
    t_int = time.perf_counter() - t0
    t_total = t_bfs + t_int * stride
    return {"value": m / t_total, "unit": UNIT, "cores": threads, "kind": "port",
            "seconds_full_extrapolated": t_total, "t_bfs_s": t_bfs,
            "t_intersect_sample_s": t_int,
            "sample": f"oracle (C restatement of the reference kernels): full BFS on 1 core "
                      f"+ CETC-SM on {threads} threads over every {stride}th edge "
                      f"({len(sub_u)} of {m}), extrapolated x{stride}"}


# ---------------------------------------------------------------------------


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; "
                         f"launch with --nproc-per-node {args.gpus} or drop torchrun")
    return world, rank, local


def spawn_ranks(args) -> int:
    """--gpus N > 1 without torchrun: start N ranks (one per GPU) with
    torch.distributed.run on 127.0.0.1; rank 0 prints the JSON line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def workload_config(name: str, n: int, m: int, ncover: int, triangles: int) -> dict:
    """The `config` dict both arms print (identical by construction)."""
    csr_bytes = 8 * (n + 1) + 8 * m
    return {"workload": name, "n": int(n), "m": int(m), "ncover": int(ncover),
            "triangles": int(triangles),
            "l2": ("inputs larger than L2" if csr_bytes >= 4 * L2_BYTES
                   else "L2 flushed between steps (GPU arm)")}


def cpu_model() -> str:
    try:
        for ln in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
            if ln.startswith("Model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args):
    """--impl reference: the reference's CPU path (the oracle's C port,
    oracle/cetc_oracle.c, of _kernels.py:129-157 and :729-755 under
    parallel.py:117-137) on the host cores, same config/metric.  Rank 0
    only.  Measured in full: timed region = 1-core BFS + CETC-SM over all m
    edges, split into K contiguous edge ranges (one per step)."""
    world, rank, _ = dist_setup(args)
    if rank != 0:
        return
    import oracle
    from paper_2403_02997_b200 import configs as C
    cfg = C.CONFIGS[args.config]
    threads = oracle.max_threads()
    t0 = time.time()
    if cfg.kind == "rmat":
        perm = C.id_permutation(cfg.n, cfg.perm_seed)
        pairs = oracle.rmat_pairs(cfg.scale, cfg.edge_factor, seed=cfg.seed, perm=perm)
    elif cfg.kind == "er":
        pairs = C.er_pairs(cfg.n, cfg.p, cfg.seed)
    else:
        pairs = C.lattice_pairs(cfg.side)
    row, nb, eu, ev = oracle.normalize(cfg.n, pairs)
    del pairs
    build_s = time.time() - t0
    m = len(eu)
    K = max(1, args.steps)
    bounds = [m * k // K for k in range(K + 1)]
    # warm-up: W short ranges (0.1% of the edges each) — thread pool, pages
    wlen = max(1, m // 1000)
    for i in range(args.warmup):
        k0 = (i * 7919 * wlen) % max(1, m - wlen)
        oracle.cetc_sm_counts(row, nb, np.zeros(cfg.n, dtype=np.int64),
                              np.ascontiguousarray(eu[k0:k0 + wlen]),
                              np.ascontiguousarray(ev[k0:k0 + wlen]), threads=threads)
    # timed: BFS (1 core, as the reference's bfs_label) + K edge ranges; a
    # run under 1 s is repeated (up to 20 runs, ~5 s) and the runs averaged
    eus = [np.ascontiguousarray(eu[bounds[k]:bounds[k + 1]]) for k in range(K)]
    evs = [np.ascontiguousarray(ev[bounds[k]:bounds[k + 1]]) for k in range(K)]

    def one_run():
        t0 = time.perf_counter()
        lev, _, comps, max_level = oracle.bfs_levels(row, nb, cfg.n)
        tb_ = time.perf_counter() - t0
        c1 = c2 = 0
        ts = []
        for k in range(K):
            t0 = time.perf_counter()
            a, b = oracle.cetc_sm_counts(row, nb, lev, eus[k], evs[k], threads=threads)
            ts.append(time.perf_counter() - t0)
            c1 += a
            c2 += b
        return tb_, ts, lev, comps, max_level, c1, c2

    runs = [one_run()]
    t_first = runs[0][0] + sum(runs[0][1])
    R = 1 if t_first >= 1.0 else min(20, max(1, int(5.0 / max(t_first, 1e-6))))
    for _ in range(R - 1):
        runs.append(one_run())
    _, _, level, comps, max_level, c1, c2 = runs[0]
    assert all(r[5:] == (c1, c2) for r in runs)
    assert c2 % 3 == 0, "c2 % 3 != 0"  # parallel.py:127-128
    T = c1 + c2 // 3
    t_bfs = float(np.mean([r[0] for r in runs]))
    step_s = [float(np.mean([r[1][k] for r in runs])) for k in range(K)]
    total = t_bfs + sum(step_s)
    value = m / total
    ncover = int(np.count_nonzero(level[eu] == level[ev]))
    sample = (f"complete run, measured: oracle (C port of the reference) 1-core BFS "
              f"{t_bfs:.2f} s + CETC-SM on {threads} threads over all {m} edges in {K} "
              f"contiguous ranges ({sum(step_s):.2f} s); no extrapolation"
              + (f"; mean of {R} complete runs" if R > 1 else ""))
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": K, "warmup": args.warmup,
            "ms_per_step": total / K * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": workload_config(cfg.name, cfg.n, m, ncover, T),
            "timed_runs": R, "seconds_full_run": total,
            "step_note": ("step k = CETC-SM over edge range k of K (BFS charged to the run); "
                          "ms_per_step = full-run time / K"),
            "counts": {"c1": c1, "c2": c2, "components": comps, "max_level": max_level},
            "host_build_s": round(build_s, 1),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "cpu_model": cpu_model(), "sample": sample,
                             "t_bfs_s": t_bfs, "t_cetc_sm_s": sum(step_s)},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        raise SystemExit(spawn_ranks(args))
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2403_02997_b200 as tb
    from paper_2403_02997_b200 import configs as C

    world, rank, local = dist_setup(args)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    cfg = C.CONFIGS[args.config]
    t0 = time.time()
    dg = C.build_device_graph(cfg, device=local)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    ctx = tb._lib.context(local)

    # L2 flush buffer for configs whose working set fits in L2
    flush = None
    if dg.nbytes < 4 * L2_BYTES:
        flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev)

    def step():
        if world > 1:  # owner-sharded intersection + one 16-byte all-reduce
            r = tb.ops.cetc_shard(dg, rank, world)
            return r, list(tb.dist.reduce_counts(r.c1, r.c2, device=dev))
        r = tb.cetc(dg)
        return r, [r.triangles, r.c1, r.c2]

    # work statistics from one labeled pass (not timed)
    full = tb.cetc(dg, keep_level=True, keep_cover=True)
    deg = (dg.row_offsets[1:] - dg.row_offsets[:-1])
    du = deg[full.cover_u.long()]
    dv = deg[full.cover_v.long()]
    W = int((du + dv).sum().item())
    W_min = int(torch.minimum(du, dv).sum().item())
    H = full.c1 + full.c2
    ncover = full.ncover
    expect = [full.triangles, full.c1, full.c2]
    # bytes the CTA-tier kernel must move (owners with d > WT = 256).  With
    # the level rule applied before the intersection (intersect.cu) an edge
    # (owner x, partner p) streams OFF(p) (p's neighbours on another level)
    # and p's same-level neighbours ranked above x (degree bucket desc, id
    # asc): 4 B/id.  Plus the partner's record per cover edge (16 B: list
    # starts, OFF size, exact UP cut, written by k_edge_prep), and the owner's
    # OFF(x) ∪ UP(x) staged once per item (<= 1024 partners).
    cu, cv = full.cover_u.long(), full.cover_v.long()
    # owner order (intersect.cu): degree bucket floor(log2 d) desc, id asc
    bk = torch.floor(torch.log2(deg.clamp(min=1).double())).long()
    bu, bv = bk[cu], bk[cv]
    own_u = (bu > bv) | ((bu == bv) & (cu < cv))
    del bu, bv
    d_own = torch.where(own_u, du, dv)
    owner = torch.where(own_u, cu, cv)
    partner = torch.where(own_u, cv, cu)
    cta = d_own > 256  # intersect.cu TCB_WT
    del cu, cv, own_u, d_own
    lev = full.level.to(dev)
    n = dg.n
    srcl = dg.src.long()
    nbl = dg.neighbors.long()
    same = lev[srcl] == lev[nbl]
    n_off = torch.bincount(srcl[~same], minlength=n)
    s_src, s_nb = srcl[same], nbl[same]
    del srcl, nbl, same, lev
    # rank: degree bucket desc, id asc (higher value = ranked higher)
    order = torch.argsort(bk * (n + 1) + (n - torch.arange(n, device=dev)))
    rk = torch.empty(n, dtype=torch.long, device=dev)
    rk[order] = torch.arange(n, device=dev)
    del order
    up = rk[s_nb] > rk[s_src]
    n_up = torch.bincount(s_src[up], minlength=n)
    keys, _ = torch.sort(s_src * n + rk[s_nb])
    row_end = torch.cumsum(torch.bincount(s_src, minlength=n), 0)
    del s_src, s_nb, up
    pc, oc = partner[cta], owner[cta]
    above = row_end[pc] - torch.searchsorted(keys, pc * n + rk[oc], right=True)
    stream_cta = int((n_off[pc].sum() + above.sum()).item())
    S_cta = int(cta.sum().item())
    staged = 0
    if S_cta:
        own_ids, per_owner = torch.unique(oc, return_counts=True)
        staged = int(((n_off + n_up)[own_ids] * ((per_owner + 1023) // 1024)).sum().item())
    W_min_cta = int(torch.minimum(du, dv)[cta].sum().item())
    b_cta = 4 * stream_cta + 16 * S_cta + 4 * staged
    del keys, pc, oc, above, row_end, n_off, n_up, rk, partner, owner, cta
    del du, dv, deg, full

    for _ in range(args.warmup):
        if flush is not None:
            flush.zero_()
        _, tot = step()
        assert tot == expect, (tot, expect)

    ctx.set_timing(True)
    stage_acc = {k: 0.0 for k in tb._lib.STAGES}
    sampler = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    launches0 = ctx.launches()
    step_ms = []
    for _ in range(args.steps):
        if flush is not None:
            flush.zero_()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        _, tot = step()
        ev1.record()
        ev1.synchronize()
        step_ms.append(ev0.elapsed_time(ev1))
        st = ctx.stage_times()
        for k in stage_acc:
            stage_acc[k] += st[k]
        assert tot == expect
    launches = ctx.launches() - launches0
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    ctx.set_timing(False)

    ms = float(np.mean(step_ms))
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    stages = {k: v / args.steps for k, v in stage_acc.items()}
    value = dg.m / (ms * 1e-3)

    # e2e through the host-buffer C entry (pinned host CSR, uploads inside;
    # at N > 1 every rank uploads its replica and the partials are
    # all-reduced, the result read back on the host)
    row_h = torch.empty(dg.n + 1, dtype=torch.int64, pin_memory=True)
    nb_h = torch.empty(2 * dg.m, dtype=torch.int32, pin_memory=True)
    row_h.copy_(dg.row_offsets)
    nb_h.copy_(dg.neighbors)
    row_np, nb_np = row_h.numpy(), nb_h.numpy()

    def e2e_step():
        if world > 1:
            r = tb.ops.cetc_host_shard(row_np, nb_np, dg.n, rank, world, device=local)
            return list(tb.dist.reduce_counts(r["c1"], r["c2"], device=dev))
        r = tb.cetc_host(row_np, nb_np, dg.n, device=local)
        return [r["triangles"], r["c1"], r["c2"]]

    for _ in range(max(1, args.warmup)):
        assert e2e_step() == expect
    torch.cuda.synchronize()
    t_e2e = []
    for _ in range(args.steps):
        if flush is not None:
            flush.zero_()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        tot = e2e_step()
        t_e2e.append(time.perf_counter() - t0)
        assert tot == expect
    t_mean = float(np.mean(t_e2e))
    if world > 1:
        t = torch.tensor([t_mean], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_mean = float(t.item())
    e2e = {"value": dg.m / t_mean, "unit": UNIT,
           "h2d_bytes_per_step": world * (8 * (dg.n + 1) + 4 * 2 * dg.m),
           "d2h_bytes_per_step": world * 120,
           "ms_per_step": t_mean * 1e3,
           "path": ("tcb_cetc_host (paper_2403_02997_b200.cetc_host): pinned host CSR"
                    if world == 1 else
                    "tcb_cetc_host_shard per rank + one all-reduce: pinned host CSR replicas")}
    del row_h, nb_h

    # e2e, drop-in variant: the reference's own call, tc_cetc(Graph), on a
    # FRESH Graph over pageable frozen numpy arrays every step (no cached
    # device copy), so the pageable upload is inside the timed region
    if world == 1:
        host_g = dg.to_host()
        for _ in range(max(1, args.warmup)):
            assert tb.tc_cetc(tb.Graph(host_g.n, host_g.m, host_g.row_offsets,
                                       host_g.neighbors, host_g.edge_u,
                                       host_g.edge_v)) == expect[0]
        t_dropin = []
        for _ in range(args.steps):
            if flush is not None:
                flush.zero_()
            g_fresh = tb.Graph(host_g.n, host_g.m, host_g.row_offsets, host_g.neighbors,
                               host_g.edge_u, host_g.edge_v)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            T_fresh = tb.tc_cetc(g_fresh)
            t_dropin.append(time.perf_counter() - t0)
            assert T_fresh == expect[0]
            del g_fresh
        td = float(np.mean(t_dropin))
        e2e["dropin"] = {"value": dg.m / td, "unit": UNIT, "ms_per_step": td * 1e3,
                         "h2d_bytes_per_step": 8 * (dg.n + 1) + 4 * 2 * dg.m,
                         "d2h_bytes_per_step": 48,
                         "path": "tc_cetc(Graph) on a fresh Graph of pageable frozen numpy "
                                 "arrays (sequential.py:164-168 call shape)"}
        del host_g

    peak, peak_kind = hbm_peak()
    # roofline of the dominant kernel, k_isect_cta (the CTA tier of the
    # intersection), timed alone with CUDA events on its launch stream
    t_cta = stages["isect_cta"] * 1e-3
    achieved = b_cta / t_cta / 1e9 if t_cta > 0 else None
    # SURVEY.md §8(d)'s merge-equivalent bytes for the whole intersection
    # stage (both lists streamed per cover edge) — above P by construction
    b_int = 4 * W + 24 * ncover + 4 * H
    t_int = stages["intersect"] * 1e-3
    b_bfs = 8 * (dg.n + 1) + 16 * dg.m + 4 * dg.n
    t_bfs = (stages["components"] + stages["bfs"]) * 1e-3
    traffic = None
    prof = ROOT / "profiles" / "ncu_traffic.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get(cfg.name, {}).get("k_isect_cta_dram_bytes")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "kernel": "k_isect_cta",
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "peak_kind": peak_kind, "algorithmic_bytes": b_cta,
                "formula": ("4*sum_{S_cta} (|OFF(p)| + |same-level N(p) ranked above x|) "
                            "+ 16*|S_cta| + 4*staged |OFF(x)|+|UP(x)| per item"),
                "stream_ids": stream_cta, "W_min_cta": W_min_cta,
                "t_ms": stages["isect_cta"],
                "survey_8d_intersect_stage": {
                    "bytes": b_int, "t_ms": stages["intersect"],
                    "effective_GBps": b_int / t_int / 1e9 if t_int > 0 else None,
                    "formula": "4*W + 24*|S| + 4*(c1+c2), W = sum_S (d(u)+d(v))"},
                "bfs": {"achieved": b_bfs / t_bfs / 1e9 if t_bfs > 0 else None,
                        "bytes": b_bfs, "t_ms": stages["components"] + stages["bfs"],
                        "formula": "8(n+1) + 16m + 4n (SURVEY.md 8(d), BFS incl. components)",
                        "frac": (b_bfs / t_bfs / 1e9 / peak) if t_bfs > 0 else None,
                        "bfs_kernel": {
                            "achieved": (b_bfs / (stages["bfs"] * 1e-3) / 1e9
                                         if stages["bfs"] > 0 else None),
                            "t_ms": stages["bfs"],
                            "frac": (b_bfs / (stages["bfs"] * 1e-3) / 1e9 / peak
                                     if stages["bfs"] > 0 else None),
                            "note": "the BFS kernels alone (k_bfs_probe + k_bfs_coop, both BFS passes)"},
                        "components_ms": stages["components"]}}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "int32", "data": "synthetic (seeded generator, see DESIGN.md)",
            "config": workload_config(cfg.name, dg.n, dg.m, ncover, expect[0]),
            "parallelism": f"replicated CSR, cover set sharded x{world}",
            "work": {"W": W, "W_min": W_min, "c1": expect[1], "c2": expect[2],
                     "graph_build_s": round(build_s, 3)},
            "stages_ms": stages, "clocks": clocks, "gpu_launches": launches,
            "e2e": e2e, "roofline": roofline}

    if rank == 0 and world == 1 and args.cpu_baseline != "off":
        import oracle
        row = dg.row_offsets.cpu().numpy()
        nb = dg.neighbors.cpu().numpy()
        eu_d, ev_d = dg.edge_arrays()
        eu, ev = eu_d.cpu().numpy(), ev_d.cpu().numpy()
        del eu_d, ev_d
        line["cpu_baseline"] = cpu_sample(dg.n, row, nb, eu, ev, args.cpu_seconds,
                                          oracle.max_threads())
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
