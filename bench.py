#!/usr/bin/env python
"""Benchmark: NNConv (edge-conditioned convolution) layer fwd+bwd edges/s on
B200 (BASELINE.json metric), DS-MPNN hot path through libdsmpnn.so.

One step = one pass of the whole hot path over one synthetic sample
(Alg. 1 :391-418): Nystrom sampling,
RCB decomposition with overlap l = r, cell-list radius graph with the n_e cap,
edge attributes, then L layers forward (each followed by the halo refresh) and
L layers backward, then the gradient sum across processes.

value = (sum over all sub-domains of E_p) * L / t_step   [edge-layers/s, fwd+bwd]

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config darcy] [--dtype bf16|f32]
    python bench.py --impl reference ...   # the CPU oracle, timed on a bounded sample

Under torchrun (N > 1) every process holds nparts/N sub-domains; halos between
processes go over NCCL (torch.distributed), timing is the max over ranks.
"""
import argparse
import dataclasses
import gc
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "NNConv layer fwd+bwd edges/sec at 1/2/4/8 B200; % tensor/HBM roofline"
UNIT = "edge-layers/s (fwd+bwd)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="darcy")
    ap.add_argument("--dtype", default=os.environ.get("DSMPNN_BENCH_DTYPE", "bf16"), choices=["bf16", "f32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=15.0)
    ap.add_argument("--streams", type=int, default=2, help="CUDA streams the local sub-domains are spread over")
    ap.add_argument("--no-comm", action="store_true",
                    help="skip every halo refresh (PAPER.md:209 no-communication ablation; halos stay stale)")
    ap.add_argument("--halo-ratio", type=float, default=1.0, help="overlap length l = ratio * r (Table 4 sweep)")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle parity check of the timed run")
    ap.add_argument("--batch", type=int, default=-1, choices=[-1, 0, 1],
                    help="sub-domains of a process as one union graph (a8): -1 auto, 0 per part, 1 on")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="build each step's graph inside the step (no prefetch of the next step's graph)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def step_config(cfg_name, world, dtype, halo_ratio=1.0, halo=True):
    from paper_2402_15106_b200 import _lib as L
    from paper_2402_15106_b200 import synth
    from paper_2402_15106_b200.api import StepConfig
    cfg = synth.CONFIGS[cfg_name]
    coords, attr = synth.points(cfg, parts=max(world, cfg.P) if cfg.kind == "weak" else None)
    n = len(coords)
    nparts = max(cfg.P, world) if cfg.kind != "weak" else world
    s = cfg.s if cfg.s else n
    sc = StepConfig(n_points=n, s=min(s, n), dim=cfg.dim, n_attr=attr.shape[1], nparts=nparts, r=cfg.r,
                    overlap_l=float(np.float32(halo_ratio * cfg.r)), n_e=cfg.n_e, halo=int(halo), d=cfg.d, k=cfg.k, L=cfg.L,
                    edge_mode=L.EDGE_DIFF if cfg.edge_mode == "diff" else L.EDGE_CONCAT,
                    dtype=L.BF16 if dtype == "bf16" else L.F32,
                    seed_sampling=synth.BASE_SEED + synth.SEED_SAMPLING,
                    seed_capping=synth.BASE_SEED + synth.SEED_CAPPING)
    return cfg, sc, coords, attr


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: an NVML
    poll thread (NVML initialised before the region, so no process start-up
    lands inside it), else an `nvidia-smi -lms 100` process."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None
        self.nv = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.bits = (pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                         pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap)
            self.max_sm = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self.nv = None

    def _poll(self):
        nv = self.nv
        while not self.done.is_set():
            try:
                sm = float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, {n for n, bit in zip(self.NAMES, self.bits) if rs & bit}))
            except Exception:
                pass
            self.done.wait(0.02)

    def start(self):
        if self.nv is not None:
            import threading
            self.samples, self.done = [], threading.Event()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.nv is not None:
            self.done.set()
            self.t.join()
            if not self.samples:
                return None
            reasons = set().union(*[r for _, r in self.samples])
            return {"sm_mhz": statistics.median([sm for sm, _ in self.samples]), "sm_max_mhz": self.max_sm,
                    "reasons": sorted(reasons), "samples": len(self.samples), "source": "nvml"}
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        out, _ = self.p.communicate()
        rows = [r.split(",") for r in out.strip().splitlines() if r.strip()]
        sm, mx, reasons = [], [], set()
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
                for nm, flag in zip(self.NAMES, r[3:7]):
                    if flag.strip() == "Active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                pass
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi"}


def count_our_launches(fn):
    """Kernels launched by one call of fn, from a CUPTI trace (torch.profiler)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    ours = other = 0
    for ev in prof.events():
        if ev.device_type.name != "CUDA":
            continue
        name = ev.name
        if "dsmpnn" in name:
            ours += 1
        elif "cub" in name.lower() and ("Radix" in name or "Scan" in name or "Sort" in name):
            other += 1
    return ours, other


def ncu_traffic(kernel, config):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` on
    `config` from the committed `ncu --set full` summary
    (profiles/ncu_traffic.json, keyed kernel -> config), or None when no
    capture of that kernel on that config is recorded (never another config's)."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")) as f:
            rec = json.load(f).get(kernel, {}).get(config)
        return (rec["bytes_per_launch"], rec.get("source")) if rec else (None, None)
    except (OSError, ValueError, KeyError, AttributeError):
        return None, None


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, \
        "fallback"


# ------------------------------------------------------------ oracle leg ---
def oracle_baseline(cfg_name, budget_s, world=1):
    """The CPU oracle as it stands, on a bounded sample of the same workload:
    layer fwd + bwd (masked upstream) for a few destination rows of the
    sampled graph, timed on this host's cores."""
    from oracle import features, graph, layer, sample
    from oracle.layer import ACT_RELU, ROOT_DENSE, LayerDesc
    from paper_2402_15106_b200 import synth
    cfg = synth.CONFIGS[cfg_name]
    coords, attr = synth.points(cfg, parts=max(world, cfg.P) if cfg.kind == "weak" else None)
    n = len(coords)
    s = cfg.s if cfg.s else n
    ids = sample.sample(n, min(s, n), synth.BASE_SEED + synth.SEED_SAMPLING)
    x, a, gid = coords[ids], attr[ids], ids.astype(np.int64)
    mode = cfg.edge_mode
    d, k = cfg.d, cfg.k
    g = np.random.default_rng(0)
    rows_all = g.permutation(len(x))
    edges = 0
    t_layer = 0.0
    done_rows = 0
    W = None
    t_start = time.perf_counter()
    for r0 in range(0, len(rows_all), 2):
        rows = np.sort(rows_all[r0:r0 + 2])
        adj = graph.radius_graph_rows(x, gid, rows, cfg.r, cfg.n_e, synth.BASE_SEED + synth.SEED_CAPPING)
        # local CSR over these destination rows, sources indexed globally
        rp = np.zeros(len(rows) + 1, np.int64)
        rp[1:] = np.cumsum([len(q) for q in adj])
        col = np.concatenate(adj).astype(np.int64)
        e = features.edge_features(mode, x, a, np.repeat(rows, np.diff(rp)), col)
        if W is None:
            W = synth.weights(e.shape[1], d, d, k)
            desc = LayerDesc(e.shape[1], d, d, k, ROOT_DENSE, ACT_RELU)
            v = synth.node_features(len(x), d)
            Gall = synth.upstream_grad(len(x), d)
        # destination rows are renumbered 0..len(rows)-1; v rows of the destinations first
        vloc = np.concatenate([v[rows], v])
        col_l = col + len(rows)
        t0 = time.perf_counter()
        layer.layer_fwd(desc, W, vloc, e, rp, col_l)
        layer.layer_bwd(desc, W, vloc, e, rp, col_l, Gall[rows])
        t_layer += time.perf_counter() - t0
        edges += int(rp[-1])
        done_rows += len(rows)
        if time.perf_counter() - t_start > budget_s:
            break
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        threads = os.cpu_count()
    return {"value": edges / t_layer, "unit": UNIT, "cores": int(threads), "kind": "oracle",
            "sample": f"{done_rows} destination rows ({edges} edges) of config '{cfg_name}', one layer fwd+bwd "
                      f"(fp64 numpy oracle, K_p materialised, masked upstream gradient); graph rows and edge "
                      f"attributes built outside the timed layer calls"}


def oracle_baseline_both(cfg_name, budget_s, world=1):
    """the oracle on all host cores (numpy's thread pool) and on
    one core, each on half the budget; `value` is the all-cores figure."""
    allc = oracle_baseline(cfg_name, budget_s / 2, world)
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1):
            one = oracle_baseline(cfg_name, budget_s / 2, world)
        allc["single_core"] = {"value": one["value"], "cores": 1, "sample": one["sample"]}
    except ImportError:
        pass
    allc["host_cpus"] = os.cpu_count()
    return allc


def oracle_parity(hp, sc, cfg_name, world, n_rows=96):
    """the benchmarked run is checked against the oracle
    after the timed region, on the same synthetic inputs (nothing the oracle
    consumes comes from the CUDA path):
      * Nystrom sample (a1): all s ids, bit-exact;
      * partition (a3): the local order of this rank's first sub-domain, bit-exact;
      * radius graph (a2): n_rows hash-selected destination rows, bit-exact;
      * layer forward (a4 + a5): layer 0 of that sub-domain on those rows,
        re-run through the same HotPath.forward the timed steps use (the
        union graph of all local sub-domains when the step runs that way);
      * layer backward (a7): layer 0 with the upstream gradient restricted to
        those rows (masked upstream), all weight gradients and dv;
    within the north_star's tolerance (1e-5 F32, 2e-2 BF16, normwise-inf)."""
    import torch
    from oracle import features, graph, layer, partition, sample
    from oracle.layer import LayerDesc
    from oracle.precision import round_bf16
    from paper_2402_15106_b200 import _lib as L
    from paper_2402_15106_b200 import synth
    t0 = time.perf_counter()
    cfg = synth.CONFIGS[cfg_name]
    coords, attr = synth.points(cfg, parts=max(world, cfg.P) if cfg.kind == "weak" else None)
    bf16 = sc.dtype == L.BF16
    tol = 2e-2 if bf16 else 1e-5
    res = {"tol": tol, "rows": n_rows}
    ids = sample.sample(sc.n_points, sc.s, sc.seed_sampling)
    res["sample_bit_exact"] = bool(np.array_equal(hp.ids.cpu().numpy(), ids))
    x_s, a_s, gid_s = coords[ids], attr[ids], ids.astype(np.int64)
    _, _, _, ranks = partition.plan(x_s, gid_s, sc.nparts, sc.overlap_l, sc.r)
    sd = hp.subs[0]
    rk = ranks[sd.rank]
    res["partition_bit_exact"] = bool(np.array_equal(sd.local_rows.cpu().numpy(), rk["local_rows"])
                                      and sd.n_deep == rk["n_deep"] and sd.n_near == rk["n_near"])
    lr = rk["local_rows"]
    x, a, gid = x_s[lr], a_s[lr], gid_s[lr]
    g = np.random.default_rng(1000 + sd.rank)
    rows = np.sort(g.choice(sd.n_own, size=min(n_rows, sd.n_own), replace=False))
    adj = graph.radius_graph_rows(x, gid, rows, sc.r, sc.n_e, sc.seed_capping)
    rph = sd.row_ptr_host.numpy()
    colg = sd.col_idx.cpu().numpy()
    res["graph_bit_exact"] = bool(all(np.array_equal(colg[rph[i]:rph[i + 1]], q) for i, q in zip(rows, adj)))
    # the oracle's CSR over the selected rows, renumbered 0..m-1 (sources: the local rows, shifted by m)
    m = len(rows)
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum([len(q) for q in adj])
    col = np.concatenate(adj).astype(np.int64)
    mode = "diff" if sc.edge_mode == L.EDGE_DIFF else "concat"
    e = features.edge_features(mode, x, a, np.repeat(rows, np.diff(rp)), col)
    W = synth.weights(e.shape[1], sc.d, sc.d, sc.k)
    v0_all = synth.node_features(sc.s, sc.d)
    G_all = synth.upstream_grad(sc.s, sc.d)
    v = v0_all[lr]
    Wo, vo, eo = dict(W), v, e
    if bf16:
        for nm in ("W1", "W2", "W3", "b3", "W_root"):
            Wo[nm] = round_bf16(W[nm])
        vo, eo = round_bf16(v), round_bf16(e)
    desc = LayerDesc(e.shape[1], sc.d, sc.d, sc.k, sc.root, sc.act, "bf16" if bf16 else "none")
    vloc = np.concatenate([vo[rows], vo])
    out_o, pre_o = layer.layer_fwd(desc, Wo, vloc, eo, rp, col + m)
    # GPU: the timed path's forward (same inputs, deterministic), layer 0 of this sub-domain
    dev = hp.dev
    v0_d = torch.from_numpy(np.ascontiguousarray(v0_all)).to(dev)
    acts, _ = hp.forward(v0_d)
    # union-graph mode (a8): sub-domain 0's owned rows are union rows [0, n_own)
    # and its halo rows start at bat.halo_off[0]
    bat = getattr(hp, "bat", None)
    if bat is not None:
        v_in, a_out, ws_f, bkey = acts[0], acts[1], hp.ws[("fwd", 0, "B")], ("bwd", "B")
        gsrc = bat
        loc_map = np.concatenate([np.arange(sd.n_own), bat.halo_off[0] + np.arange(sd.n_halo)])
    else:
        v_in, a_out, ws_f, bkey = acts[0][0], acts[1][0], hp.ws[("fwd", 0, 0)], ("bwd", 0)
        gsrc = sd
        loc_map = np.arange(sd.n_loc)
    out_g = a_out[: sd.n_own].float().cpu().numpy()[rows]
    res["fwd_err"] = _nerr(out_g, out_o)
    # masked-upstream backward of layer 0 (kinks within 2% of the spread masked, as in the tests)
    Gm = G_all[lr][rows].copy()
    if bf16 and sc.act == 1:
        Gm[np.abs(pre_o) < 2e-2 * pre_o.std()] = 0.0
    dv_o, _, g_o = layer.layer_bwd(desc, Wo, vloc, eo, rp, col + m, Gm, want_de=False)
    dv_o_full = dv_o[m:].copy()
    dv_o_full[rows] += dv_o[:m]
    Gd = torch.zeros((gsrc.n_own, sc.d), dtype=torch.float32, device=dev)
    Gd[torch.from_numpy(rows).to(dev)] = torch.from_numpy(Gm.astype(np.float32)).to(dev)
    gv = torch.zeros((gsrc.n_loc, sc.d), dtype=torch.float32, device=dev)
    grads = {n: torch.zeros_like(t) for n, t in hp.W.items()}
    ein = gsrc.e16 if bf16 else gsrc.e32
    bws = hp._ws(bkey, L.layer_bwd_workspace_size(hp.desc, gsrc.n_own, gsrc.n_loc, gsrc.n_edges))
    L.layer_bwd(hp.desc, hp.W, hp.packed, v_in, ein, gsrc.row_ptr, gsrc.col_idx, gsrc.csc_perm, gsrc.csc_ptr,
                gsrc.n_own, gsrc.n_loc, 0, gsrc.n_own, Gd, gv, None, grads, ws_f, bws,
                row_ptr_host=gsrc.row_ptr_host)
    torch.cuda.synchronize()
    errs = {"dv": _nerr(gv.cpu().numpy()[loc_map], dv_o_full)}
    for nm, t in grads.items():
        errs[nm] = _nerr(t.cpu().numpy(), g_o[nm])
    res["bwd_err_max"] = max(errs.values())
    res["bwd_err"] = errs
    res["ok"] = bool(res["sample_bit_exact"] and res["partition_bit_exact"] and res["graph_bit_exact"]
                     and res["fwd_err"] <= tol and res["bwd_err_max"] <= tol)
    res["oracle_s"] = time.perf_counter() - t0
    return res


def _nerr(x, ref):
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.abs(ref).max() if ref.size else 0.0
    return float(np.abs(x - ref).max() / den) if den > 0 else float(np.abs(x - ref).max() if x.size else 0.0)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2402_15106_b200 import synth
    cfg = synth.CONFIGS[args.config]
    per_step_budget = max(2.0, 120.0 / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        oracle_baseline(args.config, per_step_budget / 4, world)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vals.append(oracle_baseline(args.config, per_step_budget, world))
    vals[-1]["host_cpus"] = os.cpu_count()
    step_ms = (time.perf_counter() - t0) * 1e3 / max(1, args.steps)
    value = float(np.median([v["value"] for v in vals]))
    cb = dict(vals[-1])
    cb["value"] = value
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: BASELINE.json configs sample (CPU oracle, bounded)"},
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0




# -------------------------------------------------------------- our leg ----
def spawn_ranks(args):
    """`python bench.py --gpus N` (N > 1) outside a torchrun launch: start N
    ranks on this node with torch.distributed.run (127.0.0.1 rendezvous) and
    forward its exit status; rank 0 prints the line."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def f_fb_d2(subs, k, d, d_e):
    """Algorithmic fwd+bwd FLOPs of the formulation run (D2, "aggregate
    first"): per edge 6k^2 + 4 d_e k + 6(k+1) d; per
    destination row with edges 6 (k+1) d^2 (the row contraction S~ . Theta~
    forward, its two backward products)."""
    tot = 0.0
    for sd in subs:
        rp = sd.row_ptr_host.numpy()
        rows_with_edges = int((np.diff(rp) > 0).sum())
        tot += sd.n_edges * (6 * k * k + 4 * d_e * k + 6 * (k + 1) * d) + rows_with_edges * 6 * (k + 1) * d * d
    return tot


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    rank, world, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args)
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        return 2
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2402_15106_b200 import _lib as L
    from paper_2402_15106_b200 import synth
    from paper_2402_15106_b200.api import HotPath
    cfg, sc, coords, attr = step_config(args.config, world, args.dtype, args.halo_ratio, not args.no_comm)
    sc = dataclasses.replace(sc, streams=args.streams, batch=args.batch)
    d_e = (sc.dim + sc.n_attr) * (1 if sc.edge_mode == L.EDGE_DIFF else 2)
    W = synth.weights(d_e, sc.d, sc.d, sc.k)
    v0 = synth.node_features(sc.s, sc.d)
    G = synth.upstream_grad(sc.s, sc.d)
    host = {n: torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for n, a in
            (("coords", coords), ("attr", attr), ("v0", v0), ("G", G))}
    devin = {n: t.to(dev) for n, t in host.items()}
    hp = HotPath(sc, W, dev, rank, world)  # world > 1: the library NCCL context (dsmpnn_ctx_create)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2

    pipelined = not args.no_pipeline

    def step(inp, nxt=None, ready=None, serial=False):
        """One step.  Pipelined (default): the graph of this step was built
        during the previous step (HotPath.step_pipelined) and, if `nxt` is
        given, the next step's graph is built while this step's layers run.
        A run of K pipelined steps does K builds and K layer passes."""
        flush.zero_()
        if serial or not pipelined:
            return hp.step(inp["coords"], inp["attr"], inp["v0"], inp["G"])
        return hp.step_pipelined(inp["coords"], inp["attr"], inp["v0"], inp["G"],
                                 next_inputs=(nxt["coords"], nxt["attr"]) if nxt is not None else None,
                                 next_ready=ready)

    def run_steps(n, marks=None):
        """n steps of the steady-state pipeline: every step prefetches its
        successor's graph (the last warm-up step prefetches the first timed
        step's), so a timed run of K steps holds K layer passes and K builds
        (those of steps 2 .. K+1); the region ends after the last build."""
        for k_ in range(n):
            step(devin, devin if pipelined else None)
            if marks is not None and k_ < n - 1:
                marks[k_].record(torch.cuda.current_stream())

    def drop_prefetch():
        """Forget a prefetched graph (after a timed region) so the next
        region starts from a graph built from its own inputs."""
        if pipelined:
            torch.cuda.current_stream().wait_stream(hp._build_stream())
            hp._next = None

    run_steps(args.warmup)
    # settle: at least 8 untimed steps in all (W + extra) before timing; with
    # fewer, the first timed steps of a fresh process were occasionally 10-30 %
    # slow (two-stream schedule not yet steady); reported as warmup_extra
    warmup_extra = max(0, 8 - args.warmup)
    run_steps(warmup_extra)
    torch.cuda.synchronize()
    E_local = hp.n_edges
    # dominant kernel of the step: the fused edge backward (BF16), the kappa-MLP
    # second-layer GEMM (F32)
    probe_id = L.PROBE_BF16_EDGE_BWD if sc.dtype == L.BF16 else L.PROBE_F32_MLP2
    # algorithmic HBM bytes of one step's edge-backward launches (DESIGN.md
    # §6): per edge e (32 B, bf16 padded to 16) + v_j (2d) + col (4) + dz2 (2k)
    # + u_p (2d); per destination row dS_i (2(k+1)d).  The step requests no
    # edge-attribute gradient, so the kernel writes no A1 (the dW2 / dW1
    # kernels recompute a1 from e; layer_bf16_bwd.cu)
    bwd_bytes_step = sum(sd.n_edges * (32 + 4 + 4 * sc.d + 2 * sc.k) + sd.n_own * 2 * (sc.k + 1) * sc.d
                         for sd in hp.subs) * sc.L

    # ---- device-resident timed region
    # Python's cyclic GC stays off inside the timed regions (as timeit does):
    # a full collection is a host stall of tens of ms that starves the GPU of
    # launches; it runs right before each region instead
    gc.collect()
    gc.disable()
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    L.probe_begin(probe_id, 64 * args.steps * sc.L * len(hp.subs) + 64)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps - 1)]
    e0.record(st)
    run_steps(args.steps, marks)
    if pipelined:
        st.wait_stream(hp._build_stream())  # the prefetched build of step K+1 is inside the region
    e1.record(st)
    torch.cuda.synchronize()
    bounds = [e0] + marks + [e1]
    step_ms = [bounds[i].elapsed_time(bounds[i + 1]) for i in range(args.steps)]
    probe_ms, probe_n = L.probe_end()
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps

    # ---- end to end: host inputs copied in, gradients read back, every step
    out_host = {n: torch.empty_like(t, device="cpu").pin_memory() for n, t in hp.grads.items()}
    h2d = sum(t.numel() * t.element_size() for t in host.values())
    d2h = sum(t.numel() * t.element_size() for t in out_host.values())
    # inputs of step s + 1 are copied in (pinned host -> device, copy stream)
    # while step s computes; each step's gradients are staged on the device
    # (D2D) and read back on the copy stream.  Every step's copies are inside
    # the timed region, which ends when the last read-back has landed.
    cpy = torch.cuda.Stream(dev)
    dbuf = [{n: torch.empty_like(t, device=dev) for n, t in host.items()} for _ in range(2)]
    gstage = [{n: torch.empty_like(t) for n, t in hp.grads.items()} for _ in range(2)]
    loaded = [torch.cuda.Event() for _ in range(2)]
    used = [torch.cuda.Event() for _ in range(2)]

    def load_inputs(i, after=None):
        with torch.cuda.stream(cpy):
            if after is not None:
                cpy.wait_event(after)
            for n, t in host.items():
                dbuf[i][n].copy_(t, non_blocking=True)
            loaded[i].record(cpy)

    # one continuous run across calls: step s computes on dbuf[s % 2] while
    # the inputs of step s + 1 are copied into the other buffer (and, in the
    # pipeline, its graph is built from them); a call of K steps therefore
    # holds K input copies, K builds, K layer passes and K read-backs
    e2e_pos = [0]

    def e2e_run(n_steps):
        for _ in range(n_steps):
            s_ = e2e_pos[0]
            i = s_ % 2
            if s_ == 0:
                load_inputs(0)
            load_inputs(1 - i, after=used[1 - i] if s_ >= 1 else None)
            st.wait_event(loaded[i])
            grads = step(dbuf[i], dbuf[1 - i], loaded[1 - i])
            for n, t in grads.items():
                gstage[i][n].copy_(t, non_blocking=True)
            used[i].record(st)
            with torch.cuda.stream(cpy):
                cpy.wait_event(used[i])
                for n, t in gstage[i].items():
                    out_host[n].copy_(t, non_blocking=True)
            e2e_pos[0] = s_ + 1
        st.wait_stream(cpy)
        if pipelined:
            st.wait_stream(hp._build_stream())

    drop_prefetch()
    e2e_run(2)  # untimed: first use of the buffers and streams
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x0.record(st)
    e2e_run(args.steps)
    x1.record(st)
    torch.cuda.synchronize()
    e2e_ms = x0.elapsed_time(x1) / args.steps
    drop_prefetch()

    # ---- layer-only time (SURVEY D.1 t_iter: L x (fwd + halo) + L x bwd on
    # the built graphs, no graph build) with the halo exchange on and off:
    # exposed communication = t(on) - t(off) (D.4)
    def layers_ms(halo_on):
        hp.cfg = dataclasses.replace(hp.cfg, halo=int(halo_on))
        hp.forward_backward(devin["v0"], devin["G"])
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(st)
        for _ in range(args.steps):
            flush.zero_()
            hp.forward_backward(devin["v0"], devin["G"])
        a1.record(st)
        torch.cuda.synchronize()
        return a0.elapsed_time(a1) / args.steps

    layer_ms = layers_ms(sc.halo)
    layer_ms_nocomm = layers_ms(False) if sc.halo else layer_ms
    hp.cfg = dataclasses.replace(hp.cfg, halo=sc.halo)
    gc.enable()

    # roofline probe of the dominant kernel with the sub-domains on one stream:
    # with 2 streams its launches overlap other kernels, so their event
    # durations measure the schedule, not the kernel (both are reported)
    # (with the pipeline, the next step's graph build overlaps it the same way)
    probe_ms_step, probe_n_step = probe_ms, probe_n
    serial_ms = None
    if sc.streams > 1 or pipelined:
        hp.cfg = dataclasses.replace(hp.cfg, streams=1)
        step(devin, serial=True)
        torch.cuda.synchronize()
        L.probe_begin(probe_id, 64 * args.steps * sc.L * len(hp.subs) + 64)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(st)
        for _ in range(args.steps):
            step(devin, serial=True)
        s1.record(st)
        torch.cuda.synchronize()
        probe_ms, probe_n = L.probe_end()
        serial_ms = s0.elapsed_time(s1) / args.steps
        hp.cfg = dataclasses.replace(hp.cfg, streams=sc.streams)
    # kernels of one step (CUPTI trace); after the timed regions so that no
    # profiler state is live while they run
    launches, lib_other = count_our_launches(lambda: step(devin, serial=True))

    # ---- graph build alone (sample + partition + radius graph + attributes + CSC), for reference
    torch.cuda.synchronize()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    L.graph_stats(reset=True)
    g0.record(st)
    for _ in range(args.steps):
        hp.build(devin["coords"], devin["attr"])
    g1.record(st)
    torch.cuda.synchronize()
    graph_ms = g0.elapsed_time(g1) / args.steps
    graph_tests = L.graph_stats(reset=True) / args.steps  # candidate tests per build (this rank)
    # SURVEY D.3 a2 algorithmic bytes per sub-domain: n_loc (4 dim + 8) + 8 (n_dst + 1) + 4 E
    graph_bytes = sum(sd.n_loc * (4 * sc.dim + 8) + 8 * (sd.n_own + 1) + 4 * sd.n_edges for sd in hp.subs)

    stats = torch.tensor([ms, e2e_ms, layer_ms, layer_ms_nocomm, float(E_local)], dtype=torch.float64, device=dev)
    if world > 1:
        mx = stats[:4].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        tot = stats[4:].clone()
        dist.all_reduce(tot)
        stats = torch.cat([mx, tot])
    ms, e2e_ms, layer_ms, layer_ms_nocomm, E_tot = [float(x) for x in stats]
    # the formulation's own algorithmic FLOPs, summed over ranks
    fl = torch.tensor([f_fb_d2(hp.subs, sc.k, sc.d, d_e) * sc.L], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(fl)
    fl_tot = float(fl[0])
    value = E_tot * sc.L / (ms / 1e3)
    e2e_value = E_tot * sc.L / (e2e_ms / 1e3)

    parity = None
    if rank == 0 and not args.no_parity:
        parity = oracle_parity(hp, sc, args.config, world)

    if rank == 0:
        peaks, src = measured_peaks()
        k, d = sc.k, sc.d
        bwd_flops_edge = 2 * (16 * k + k * k) + 2 * 2 * k * d  # recomputed MLP + dH^T + U
        if sc.dtype == L.BF16:
            # fused edge backward: HBM-bound (its byte floor exceeds its tensor floor)
            unit, bound, peak = "GB/s", "hbm", float(peaks["hbm_gbs"])
        else:
            # F32: the kappa-MLP second layer (fp32 SIMT FFMA); peak from unit counts
            flops_edge = 2 * k * k
            unit, bound = "TFLOP/s", "alu"
            peak = 148 * 128 * 2 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
        per_launch_ms = probe_ms / max(1, probe_n)
        units_per_launch = E_local * args.steps * sc.L / max(1, probe_n)
        traffic = traffic_src = None
        if sc.dtype == L.BF16:
            bytes_per_launch = bwd_bytes_step * args.steps / max(1, probe_n)
            achieved = bytes_per_launch / (per_launch_ms / 1e3) / 1e9 if probe_n else 0.0
            tensor_tflops = bwd_flops_edge * units_per_launch / (per_launch_ms / 1e3) / 1e12 if probe_n else 0.0
            if world == 1 and args.halo_ratio == 1.0:
                traffic, traffic_src = ncu_traffic("edge_bwd4", args.config)
        else:
            achieved = flops_edge * units_per_launch / (per_launch_ms / 1e3) / 1e12 if probe_n else 0.0
            bytes_per_launch, tensor_tflops = None, None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak" if cfg.kind == "weak" else "strong", "vs_baseline": None,
            "dtype": "bf16" if sc.dtype == L.BF16 else "f32", "data": "synthetic",
            "config": {"workload": f"{cfg.name} (BASELINE.json configs[{list(synth.CONFIGS).index(cfg.name)}])",
                       "n_points": sc.n_points, "sampled": sc.s, "subdomains": sc.nparts, "radius": sc.r,
                       "overlap_l": sc.overlap_l, "halo_ratio": args.halo_ratio, "halo": "on" if sc.halo else "off",
                       "n_e": sc.n_e, "width": sc.d, "ker_width": sc.k, "layers": sc.L,
                       "edges_total": int(E_tot), "edge_attr_dim": d_e,
                       "form": "GNO: relu(W v_i + mean kappa(e) v_j + b)",
                       "l2": "256 MB buffer zeroed at the start of every step, inside the timed region",
                       "step": "sample + partition + radius graph + edge attrs + L x (fwd + halo) + L x bwd",
                       "streams": sc.streams,
                       "subdomain_batch": ("one union graph (a8)" if getattr(hp, "bat", None) is not None
                                           else "per sub-domain"),
                       "pipeline": ("the graph of step t+1 is built on a second stream while step t's layers run "
                                    "(Alg. 1 builds graphs ahead of the training loop); the timed K steps hold K "
                                    "layer passes and K builds (steps 2..K+1; step 1's graph was prefetched by the "
                                    "last warm-up step) and end after the last build"
                                    if pipelined else "off: each step builds its graph first"),
                       "comm": "library NCCL context (dsmpnn_halo_exchange)" if world > 1 else
                               "sub-domains on one device: halo = device copies"},
            "roofline": {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
                         "frac": achieved / peak if peak else None, "traffic": traffic,
                         "traffic_source": traffic_src,
                         "kernel": {1: "F32 mlp2 sgemm", 5: "bf16 fused edge bwd (edge_bwd4)"}.get(probe_id,
                                                                                               str(probe_id)),
                         "algorithmic_bytes_per_launch": bytes_per_launch,
                         "tensor_tflops_same_launches": tensor_tflops,
                         "tensor_frac": (tensor_tflops / float(peaks["bf16_tflops_sustained"])
                                         if tensor_tflops else None),
                         "per_launch_ms": per_launch_ms, "launches": probe_n,
                         "share_of_step": probe_ms / (ms * args.steps), "peak_source": src,
                         "probe": ("separate pass of the same steps, unpipelined, sub-domains on one stream "
                                   "(the kernel alone); in the timed region its launches overlap the next "
                                   "step's graph build / other streams" if (sc.streams > 1 or pipelined)
                                   else "timed region"),
                         "per_launch_ms_in_timed_region": probe_ms_step / max(1, probe_n_step)},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_ms},
            "graph_ms": graph_ms,
            "graph": {"ms": graph_ms, "candidate_tests": graph_tests,
                      "candidate_tests_per_s": graph_tests / (graph_ms / 1e3),
                      "scan_GBps": graph_tests * 16 / (graph_ms / 1e3) / 1e9,
                      "algorithmic_GBps": graph_bytes / (graph_ms / 1e3) / 1e9,
                      "what": "whole build (sample + partition + radius graph + attributes + CSC) on rank 0; "
                              "candidate tests = fp32 predicate evaluations of the radius-graph search (first pass), "
                              "16 B (cell-ordered float4) read per test; algorithmic bytes per SURVEY D.3 a2"},
            "layers_only": {"ms": layer_ms, "value": E_tot * sc.L / (layer_ms / 1e3),
                            "ms_no_comm": layer_ms_nocomm,
                            "exposed_comm_ms": layer_ms - layer_ms_nocomm if sc.halo else None,
                            "what": "L x (fwd + halo) + L x bwd on the built graphs (SURVEY D.1 t_iter), "
                                    "max over ranks; no-comm = the same with every halo refresh skipped"},
            "step_ms_min_median_max": [min(step_ms), statistics.median(step_ms), max(step_ms)],
            "step_ms": [round(x, 3) for x in step_ms],
            "ms_per_step_unpipelined": serial_ms,
            "gpu_launches": launches * args.steps,
            "warmup_extra": warmup_extra,
            "gpu_launches_cub": lib_other * args.steps,
            "clocks": clk,
        }
        if sc.dtype == L.BF16:
            line["roofline"]["d2_flops_per_step"] = fl_tot
            line["roofline"]["d2_tensor_frac_layers"] = fl_tot / (layer_ms / 1e3) / 1e12 / float(
                peaks["bf16_tflops_sustained"]) / world
            line["roofline"]["d2_tensor_frac_step"] = fl_tot / (ms / 1e3) / 1e12 / float(
                peaks["bf16_tflops_sustained"]) / world
            line["roofline"]["d2_note"] = ("F_fb(D2) = 6k^2 + 4 d_e k + 6(k+1)d per edge + 6(k+1)d^2 per row "
                                           "with edges (SURVEY D.3), / bf16_tflops_sustained; layers = graph "
                                           "build excluded, step = included")
        if parity is not None:
            line["parity"] = parity
            if not parity["ok"]:
                line["value"] = None
                line["e2e"]["value"] = None
                line["failed"] = "parity check of the timed run against the oracle failed"
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = oracle_baseline_both(args.config, args.cpu_budget_s, world)
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
