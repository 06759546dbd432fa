#!/usr/bin/env python
"""Benchmark of the matrix-free SIPG operator y = A z (arXiv 1711.10885) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload NAME]

One step = one dg_apply (the whole hot path: volume, interior-face and
boundary-face terms, plus the face-trace halo exchange when N > 1) over the
workload's synthetic seeded input already resident in HBM. At N = 1 the workload
is BASELINE.json configs[2] ("C3": 128x64x64 cells, k = 7, 268M DOFs). For N > 1
(one rank per GPU, NCCL; `python bench.py --gpus N` launches the ranks itself
through torch.distributed.run when WORLD_SIZE is unset) the default is
BASELINE configs[4]'s weak scaling, 128x128x64 cells per GPU (C5 weak), block-
partitioned 2x1x1 / 2x2x1 / 2x2x2; `--workload c5strong` is its strong scaling
(256x128x128 cells in total).

Rank 0 prints ONE JSON line. `value` is whole-job DOFs/s (max-over-ranks device
time of K steps, CUDA events, barrier + synchronize on both sides); `e2e` is the
same metric through the C ABI with pinned HOST buffers (dg_apply_host: H2D of z,
apply, D2H of y inside the timed region); `roofline` is the operator kernel's
EXECUTED FP64 rate (ncu flop count of this build x DOFs / kernel time) against
the derived B200 FP64 peak (the paper-model rate is `model_tflops`);
`cpu_baseline` is the oracle O-1 timed on the host cores on a bounded sample of
cells (N = 1, rank 0). `--impl reference` times that oracle as the reference arm.
"""
import argparse
import dataclasses
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1711_10885_b200 import configs, inputs, perfmodel  # noqa: E402

METRIC = "DOFs/s & FP64 GFLOP/s of matrix-free DG apply (k=7), % of roofline, 1/2/4/8 GPU"
UNIT = "DOF/s"


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def workload(name, world):
    if name in (None, "", "default"):
        return configs.c3() if world == 1 else configs.c5_weak(world)
    name = name.lower()
    if name == "c3weak":
        return configs.c3_weak(world)
    if name == "c5weak":
        return configs.c5_weak(world)
    if name == "c5strong":
        grid = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}[world]
        return configs.c5_strong(grid)
    if name.startswith("a-k"):
        return configs.problem_a(int(name[3:]), world)
    if name.startswith("tg-k") and world == 1:
        return configs.taylor_green(int(name[4:]))
    if name.startswith("c-k"):
        return configs.problem_c(int(name[3:]), world)
    cfg = configs.by_name(name)
    if world != 1:
        raise SystemExit("workload %s is single-GPU" % name)
    return cfg


def workload_desc(cfg, world):
    dtxt = ("per-cell SPD tensor field (inputs.tensor_field_*, seed %d)" % cfg.dfield_seed
            if cfg.dfield_seed >= 0 else str(list(cfg.D)))
    bc = "periodic" if all(cfg.periodic) else ("Dirichlet" if not any(cfg.periodic) else "periodic %s" % (cfg.periodic,))
    if cfg.bkind:
        bc += ", b(x) = Taylor-Green field at every quadrature point" if cfg.bkind == 1 else ", b(x) linear field"
    if cfg.geo_amp > 0:
        bc += (", multilinear mesh: vertices moved by <= %g h per direction (inputs.vertex_grid, seed %d)"
               % (cfg.geo_amp, cfg.geo_seed))
    if cfg.m and cfg.m != cfg.k + 1:
        bc += ", m = %d Gauss points per direction (q = %d)" % (cfg.m, 2 * cfg.m - 1)
    return {"workload": "%s: %dx%dx%d cells, k=%d, %d DOFs, box %s-%s, D=%s, b=%s, c=%g, sigma=%g, %s, seed %d"
                        % (cfg.name, cfg.ncells[0], cfg.ncells[1], cfg.ncells[2], cfg.k, cfg.ndofs,
                           list(cfg.lo), list(cfg.hi), dtxt, list(cfg.b), cfg.c, cfg.sigma, bc, cfg.seed),
            "k": cfg.k, "ncells": list(cfg.ncells), "ndofs": cfg.ndofs, "parts": list(cfg.parts),
            "parallelism": "block %dx%dx%d" % tuple(cfg.parts) if world > 1 else "1 GPU",
            "l2": "no flush: z and y are %.2f GB each per GPU (> 126 MB L2)" % (cfg.ndofs / world * 8 / 1e9)}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (B200_PROFILING.md)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def sample_cells(cfg, count, seed=0):
    """Seeded random cells plus every boundary type (corners, edges, faces, interior)."""
    rng = np.random.default_rng(seed)
    nx, ny, nz = cfg.ncells
    special = [x + nx * (y + ny * z) for x in (0, nx // 2, nx - 1) for y in (0, ny // 2, ny - 1)
               for z in (0, nz // 2, nz - 1)]
    extra = rng.integers(0, cfg.ncell, max(0, count - len(special)))
    return np.unique(np.r_[special, extra]).astype(np.int64)[:max(count, 1)]


def oracle_kw(cfg):
    """periodic / per-cell tensor / velocity / quadrature keywords of the oracle for this workload."""
    kw = {"periodic": cfg.periodic, "bkind": cfg.bkind, "m": cfg.m}
    if cfg.dfield_seed >= 0:
        kw["Dcell"] = inputs.tensor_field_cells(np.arange(cfg.ncell), cfg.dfield_seed)
    return kw


def cpu_oracle_rate(cfg, z_host, budget_s, seed=0):
    """O-1 (oracle, as it stands) on a bounded sample of cells; returns (DOF/s, cores, sample text, seconds)."""
    from oracle import o1   # only bench.py's cpu_baseline / reference legs may touch oracle/
    kw = oracle_kw(cfg)
    probe = sample_cells(cfg, 512, seed)    # large enough to amortise the thread start-up
    o1.apply(*cfg.args(), z_host, cells=probe[:32], **kw)
    t0 = time.perf_counter()
    _, cores = o1.apply(*cfg.args(), z_host, cells=probe, **kw)
    dt = max(time.perf_counter() - t0, 1e-6)
    per_cell = dt / probe.size
    count = int(min(max(budget_s / per_cell, 16), cfg.ncell))
    cells = sample_cells(cfg, count, seed + 1)
    t0 = time.perf_counter()
    yo, cores = o1.apply(*cfg.args(), z_host, cells=cells, **kw)
    dt = time.perf_counter() - t0
    rate = cells.size * cfg.n3 / dt
    text = ("O-1 naive quadrature (C/OpenMP, -O3) on %d of %d cells of %s (seeded random + all boundary types); "
            "%.1f s on %d threads of %s" % (cells.size, cfg.ncell, cfg.name, dt, cores, cpu_model()))
    return rate, cores, text, dt, cells, yo


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown CPU"


def load_ncu(cfg, kname):
    """The committed ncu --set full summary of this workload's operator kernel, or ({}, why).
    Only a capture of THIS build (paper_1711_10885_b200.build.kernel_hash) and of the same kernel
    and per-rank DOF count is used; at N > 1 the N = 1 capture of the same per-GPU block."""
    from paper_1711_10885_b200.build import kernel_family, kernel_hash
    path = os.path.join(ROOT, "profiles", "ncu_full_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
    except Exception as e:  # noqa: BLE001
        return {}, "no ncu summary (%s)" % e
    name = cfg.name.replace("-P%d" % (cfg.parts[0] * cfg.parts[1] * cfg.parts[2]), "-P1") \
        if cfg.name.startswith("C5-weak") else cfg.name
    ent = d.get(name)
    if not ent:
        return {}, "no ncu capture of %s" % name
    want = kernel_hash(kernel_family(kname))
    if ent.get("build_hash") != want:
        return {}, "ncu capture of %s belongs to build %s, not %s" % (name, ent.get("build_hash"), want)
    if kname.split("<")[0] not in ent.get("kernel", ""):
        return {}, "ncu capture of %s is of %s" % (name, ent.get("kernel"))
    return ent, "profiles/ncu_full_summary.json[%s] (ncu --set full, --clock-control none, build %s)" % (
        name, ent["build_hash"])


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def fp64_measured():
    """The builder's FP64 microbenchmarks on this pool's B200 (profiles/r01_fp64_peaks.json)."""
    out = {}
    try:
        with open(os.path.join(ROOT, "profiles", "r01_fp64_peaks.json")) as f:
            for line in f:
                line = line.strip()
                if not line:
                    continue
                d = json.loads(line)
                if d.get("kernel") == "dfma":
                    out["dfma"] = d["tflops"]
                elif "DGEMM" in d.get("kernel", ""):
                    out["dgemm"] = d["tflops_best"]
    except Exception:
        pass
    return out


def submesh_parity(cfg, op, y, rank, dev, count=6):
    """Partition invariance on this run's own output (SURVEY 8(e) evidence 4), with the product
    path only: for sampled cells of this rank -- one next to every partition face, the rest
    random -- a SINGLE-rank operator on the (up to) 3x3x3-cell sub-box around the cell (same h,
    coefficients and sigma; a clipped side is the global Dirichlet boundary) applied to the same
    seeded z (inputs.uniform_cells by global cell index) must reproduce the cell's y block.
    Returns (cells checked, max |dy| / max |y_sub|, bitwise)."""
    import torch
    from paper_1711_10885_b200 import dg
    if any(cfg.periodic) or cfg.dfield_seed >= 0 or cfg.bkind:
        return 0, None, None
    G, n3 = cfg.ncells, cfg.n3
    h = [(cfg.hi[q] - cfg.lo[q]) / G[q] for q in range(3)]
    lo, cnt = op.cell_lo, op.cell_cnt
    rng = np.random.default_rng(1000 + rank)
    picks = []
    for f in range(6):
        if op.halo_info(f)[0] < 0:
            continue
        q, sd = f >> 1, f & 1
        l = [int(rng.integers(0, cnt[r])) for r in range(3)]
        l[q] = cnt[q] - 1 if sd else 0
        picks.append(l)
    while len(picks) < count:
        picks.append([int(rng.integers(0, cnt[r])) for r in range(3)])
    worst, bitwise = 0.0, True
    yv = y.view(-1, n3)
    for l in picks:
        g = [lo[r] + l[r] for r in range(3)]
        slo = [max(0, g[r] - 1) for r in range(3)]
        shi = [min(G[r], g[r] + 2) for r in range(3)]
        sc = [shi[r] - slo[r] for r in range(3)]
        sub = dg.Operator(sc, [cfg.lo[r] + slo[r] * h[r] for r in range(3)],
                          [cfg.lo[r] + shi[r] * h[r] for r in range(3)], cfg.k, cfg.D, cfg.b, cfg.c, cfg.sigma,
                          device=dev.index)
        gz, gy, gx = np.meshgrid(np.arange(slo[2], shi[2]), np.arange(slo[1], shi[1]), np.arange(slo[0], shi[0]),
                                 indexing="ij")
        cells = (gx + G[0] * (gy + G[1] * gz)).reshape(-1)
        zs = torch.from_numpy(inputs.uniform_cells(cells, n3, cfg.seed).reshape(-1)).to(dev)
        ys = torch.empty_like(zs)
        sub.apply(zs, ys)
        mid = (g[0] - slo[0]) + sc[0] * ((g[1] - slo[1]) + sc[1] * (g[2] - slo[2]))
        a = ys.view(-1, n3)[mid]
        b = yv[l[0] + cnt[0] * (l[1] + cnt[1] * l[2])]
        worst = max(worst, float((a - b).abs().max() / ys.abs().max()))
        bitwise = bitwise and bool(torch.equal(a, b))
        sub.close()
    return len(picks), worst, bitwise


def vs_baseline(cfg, value):
    """value / the paper's number for the SAME workload: only Problem A has one (Table 1)."""
    if cfg.dfield_seed >= 0 and all(cfg.periodic) and cfg.k in perfmodel.PAPER_TABLE1_A_MDOFS:
        return value / (perfmodel.PAPER_TABLE1_A_MDOFS[cfg.k] * 1e6)
    return None


# ------------------------------------------------------------------------------------------ reference
def run_reference(args, rank, world):
    if rank != 0:
        return 0
    from oracle import o1
    gcfg = workload(args.workload, world)
    cfg = gcfg
    if world > 1:
        # the oracle is a single-host program: time one GPU-share of the workload -- rank 0's block of
        # the partition as a standalone mesh (same cells, coefficients and penalty; the per-cell cost
        # does not depend on the mesh size), instead of seeding the whole global z on the host
        # (4.3e9 doubles = 34 GB for C5 weak at N = 8)
        parts = gcfg.parts
        nloc = tuple(-(-gcfg.ncells[q] // parts[q]) for q in range(3))
        hi = tuple(gcfg.lo[q] + (gcfg.hi[q] - gcfg.lo[q]) * nloc[q] / gcfg.ncells[q] for q in range(3))
        cfg = dataclasses.replace(gcfg, name=gcfg.name + " (rank 0 block)", ncells=nloc, hi=hi, parts=(1, 1, 1))
    o1.build()
    z = inputs.uniform(cfg.ndofs, cfg.seed)
    kw = oracle_kw(cfg)
    budget = args.ref_seconds / max(1, args.steps + args.warmup)
    probe = sample_cells(cfg, 8, 0)
    t0 = time.perf_counter()
    o1.apply(*cfg.args(), z, cells=probe, **kw)
    per_cell = max(time.perf_counter() - t0, 1e-6) / probe.size
    count = int(min(max(budget / per_cell, 8), cfg.ncell))
    cells = sample_cells(cfg, count, 1)
    cores = 0
    for _ in range(args.warmup):
        _, cores = o1.apply(*cfg.args(), z, cells=cells, **kw)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        _, cores = o1.apply(*cfg.args(), z, cells=cells, **kw)
    dt = time.perf_counter() - t0
    rate = args.steps * cells.size * cfg.n3 / dt
    sample = ("each step: O-1 naive quadrature (C/OpenMP) on %d of %d cells of %s (seeded random + all boundary "
              "types)" % (cells.size, cfg.ncell, cfg.name))
    out = {"impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded splitmix64, C-13)",
           "config": workload_desc(gcfg, world),
           "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "gpu_launches": 0}
    print(json.dumps(out), flush=True)
    return 0


# ------------------------------------------------------------------------------------------ ours
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_1711_10885_b200 import dg

    # --share-gpu (development / CI on a one-GPU box): all ranks on the visible GPUs round-robin,
    # torch.distributed over gloo, no NCCL communicator (ncclCommInitRank refuses two ranks on one
    # device), the direct IPC halo; every cross-rank dependency is a stream wait on a recorded event,
    # no kernel waits on another rank (B200_PROFILING.md). Exercises the whole N-rank path; its
    # timing is N ranks time-sharing one GPU, not a scaling number.
    shared = bool(args.share_gpu) and world > 1
    gpu = local_rank % max(1, torch.cuda.device_count()) if shared else local_rank
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    red_dev = torch.device("cpu") if shared else dev   # device of the reduction tensors (gloo: host)
    cfg = workload(args.workload, world)
    if shared and args.halo != "p2p":
        raise SystemExit("--share-gpu runs the direct IPC halo only (no NCCL communicator)")
    nccl_id = None
    if world > 1 and not shared:
        idt = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            idt.copy_(torch.tensor(list(dg.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nccl_id = bytes(idt.cpu().tolist())
    op = dg.Operator(cfg.ncells, cfg.lo, cfg.hi, cfg.k, cfg.D, cfg.b, cfg.c, cfg.sigma, device=gpu, rank=rank,
                     nranks=world, parts=cfg.parts, nccl_id=nccl_id, bc=dg.bc_from_periodic(cfg.periodic))
    if cfg.dfield_seed >= 0:
        op.set_tensor_field(cfg.dfield_seed)
    if cfg.bkind:
        op.set_velocity(cfg.bkind)
    if cfg.geo_amp > 0:
        op.set_geometry(dg.padded_vertex_grid(cfg, op.cell_lo, op.cell_cnt), cfg.m or cfg.k + 1)
    elif cfg.m and cfg.m != cfg.k + 1:
        op.set_quadrature(cfg.m)
    general = cfg.dfield_seed >= 0 or any(cfg.D[i] != 0 for i in (1, 2, 3, 5, 6, 7))
    if cfg.geo_amp > 0:
        kname = "dg_geo_kernel<%d,%d>" % (cfg.k + 1, cfg.m or cfg.k + 1)
    elif cfg.bkind or (cfg.m and cfg.m != cfg.k + 1):
        kname = "dg_vb_kernel<%d,%d>" % (cfg.k + 1, cfg.m or cfg.k + 1)
    else:
        kname = "dg_gen_kernel<%d>" % (cfg.k + 1) if general else "dg_cell_kernel<%d>" % (cfg.k + 1)
    halo_note = None
    if world > 1 and args.halo == "p2p":
        # the fused halo: each rank's trace pack kernel stores into the neighbours' receive buffers
        # over NVLink (CUDA IPC); NCCL stays for setup-time exchanges and is the fallback
        try:
            dg.p2p_attach(op)
        except Exception as e:  # noqa: BLE001 -- reported in the JSON line, NCCL carries on
            if shared:
                raise
            halo_note = "direct halo unavailable (%s): NCCL send/recv" % e
        if shared:
            halo_note = ("--share-gpu: %d ranks time-share %d GPU(s); the timing is not a scaling number"
                         % (world, torch.cuda.device_count()))
    info = op.kernel_info()
    transport, comm_ranks = op.comm_info()
    if world > 1 and rank == 0:
        print("[bench] halo transport %s: communicator of %d ranks (torch.distributed world %d)"
              % (transport, comm_ranks, world), file=sys.stderr, flush=True)
    z = torch.empty(op.ndofs, dtype=torch.float64, device=dev)
    y = torch.empty_like(z)
    op.fill_uniform_local(z, cfg.seed)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(args.warmup, 3)):
        op.apply(z, y)
    torch.cuda.synchronize()

    clocks = ClockSampler(gpu)
    clocks.start()
    time.sleep(0.2)
    # ---- timed region: K steps, device time by CUDA events on the launching stream
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("timed region: %d x dg_apply" % args.steps)
    e0.record(stream)
    for _ in range(args.steps):
        op.apply(z, y)
    e1.record(stream)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    barrier()
    t_local = e0.elapsed_time(e1) * 1e-3
    # kernel-only time (no halo exchange; identical to the step at N = 1)
    if world > 1:
        k0 = torch.cuda.Event(enable_timing=True)
        k1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        k0.record(stream)
        for _ in range(args.steps):
            op.apply(z, y, terms=dg.ALL | dg.HALO_EXTERNAL)
        k1.record(stream)
        torch.cuda.synchronize()
        tk_local = k0.elapsed_time(k1) * 1e-3
    else:
        tk_local = t_local
    clk = clocks.stop()
    # overlap evidence: one armed apply's launch timeline per rank (dg_timeline)
    timeline = None
    if world > 1:
        op.timeline_arm()
        op.apply(z, y)
        tl = op.timeline()
        gathered = [None] * world
        dist.all_gather_object(gathered, tl)
        timeline = {"ms_since_apply_start": gathered,
                    "pack_hidden_in_inner": [g["pack_end"] <= g["inner_end"] for g in gathered],
                    "what": "one apply after the timed region: the trace pack (+ exchange) on the comm stream "
                            "against the inner-box kernel on the compute stream, and the shell kernel after "
                            "the received traces (CUDA events, dg_timeline)"}
    # per-step distribution (separate, after the timed region): median / min of single applies
    step_ms = []
    if world == 1:
        for _ in range(min(args.steps, 20)):
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            op.apply(z, y)
            s1.record(stream)
            s1.synchronize()
            step_ms.append(s0.elapsed_time(s1))
    t = t_local
    tk = tk_local
    if world > 1:
        tt = torch.tensor([t_local, tk_local], dtype=torch.float64, device=red_dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t, tk = float(tt[0]), float(tt[1])
    total_dofs = cfg.ndofs   # whole job (all ranks)
    value = total_dofs * args.steps / t
    ms_per_step = t / args.steps * 1e3

    # ---- roofline of the dominant kernel (the fused operator kernel): EXECUTED FP64 flops of this
    # build (ncu) per launch / the kernel's time per apply, against the FP64 peak derived from the
    # unit counts and clock (B200_PROFILING.md: 148 SMs; 64 FP64 FMA/clk/SM; clocks.max.sm)
    per_dof = perfmodel.flopdof(3, cfg.k)
    kern_t = tk / args.steps   # one operator pass over all local cells per apply (inner + shell at N > 1)
    smax = clk["sm_max_mhz"] or 1965.0
    peak = perfmodel.fp64_peak_tflops(smax)
    meas = fp64_measured()
    ncu, ncu_src = load_ncu(cfg, kname)
    try:
        hbm_peak = float(measured_peaks().get("hbm_gbs"))      # MEASURED_PEAKS.json copy bandwidth
    except (TypeError, ValueError):
        hbm_peak = None
    exec_per_dof = ncu.get("executed_flops_per_dof")
    traffic = ncu.get("dram_bytes_per_launch")
    achieved = exec_per_dof * op.ndofs / kern_t / 1e12 if exec_per_dof else None
    model_tf = per_dof * op.ndofs / kern_t / 1e12
    roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak if achieved else None,
            "traffic": traffic,
            "flops_basis": ("executed FP64 flops of this build: ncu 2 DFMA + DADD + DMUL = %.1f flop/DOF x %d DOFs "
                            "per apply" % (exec_per_dof, op.ndofs)) if exec_per_dof else
                           ("unavailable: %s" % ncu_src),
            "peak_basis": "derived: 148 SMs x 64 FP64 FMA/clk x 2 x %.0f MHz (MEASURED_PEAKS.json has no FP64 "
                          "entry; B200_PROFILING.md unit counts)" % smax,
            "frac_of_measured_dfma": achieved / meas["dfma"] if (achieved and "dfma" in meas) else None,
            "frac_of_measured_dgemm": achieved / meas["dgemm"] if (achieved and "dgemm" in meas) else None,
            "measured_fp64_tflops": dict(meas, source="profiles/r01_fp64_peaks.json (tools/fp64_peaks.cu, "
                                                       "torch float64 matmul)"),
            "model_tflops": model_tf, "model_frac": model_tf / peak,
            "model_basis": "paper model FLOPDOF_vol + FLOPDOF_face(3,%d) = %.1f flop/DOF (PAPER.md:675-676); the "
                           "kernel executes fewer (collocation derivatives, even-odd stages), so model_frac can "
                           "exceed 1" % (cfg.k, per_dof),
            "traffic_algorithmic_bytes": 16.0 * op.ndofs,
            "hbm_gbs_at_traffic": (traffic / kern_t / 1e9) if traffic else None,
            "hbm_frac_of_measured_copy": (traffic / kern_t / 1e9 / hbm_peak) if (traffic and hbm_peak) else None,
            "ncu_fp64_pipe_pct": ncu.get("fp64_pipe_pct"), "ncu_smem_wavefront_pct": ncu.get("smem_wavefront_pct"),
            "ncu_issue_active_pct": ncu.get("issue_active_pct"),
            "ncu_source": ncu_src,
            "kernel": "%s (FP64 DFMA pipe)" % kname,
            "kernel_ms": kern_t * 1e3}

    # ---- end to end through the C ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        zh = z.cpu().pin_memory().numpy()
        yh = torch.empty(op.ndofs, dtype=torch.float64).pin_memory().numpy()
        op.apply_host(zh, yh)   # warm (allocates the device staging once)
        ke = max(2, min(args.steps, args.e2e_steps))
        barrier()
        t0 = time.perf_counter()
        for _ in range(ke):
            op.apply_host(zh, yh)
        te = time.perf_counter() - t0
        if world > 1:
            tt = torch.tensor([te], dtype=torch.float64, device=red_dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt[0])
        e2e = {"value": total_dofs * ke / te, "unit": UNIT, "h2d_bytes_per_step": op.ndofs * 8 * world,
               "d2h_bytes_per_step": op.ndofs * 8 * world, "steps": ke,
               "path": "dg_apply_host (pinned host z; z-slab pipeline: H2D / fused kernel / D2H overlapped on 3 streams), wall clock, max over ranks"}

    # ---- CPU baseline: the oracle on the host cores (rank 0, N = 1 only)
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and cfg.geo_amp > 0:
        cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "oracle",
               "sample": "not timed: the multilinear-geometry oracle (oracle/o2_geometry.py) assembles dense "
                         "matrices on tiny meshes only"}
    elif rank == 0 and world == 1 and not args.no_cpu_baseline:
        zn = z.cpu().numpy()
        rate, cores, text, _, cells, yo = cpu_oracle_rate(cfg, zn, args.cpu_seconds)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": "extrapolated: DOF/s measured on a sample -- " + text}
        # the same oracle blocks double as a parity check of this run's y (reading C-14)
        yg = y.view(-1, cfg.n3)[torch.from_numpy(cells).to(dev)].cpu().numpy()
        ymax = float(y.abs().max())
        parity = {"vs": "O-1 on the cpu_baseline sample (%d cells)" % cells.size,
                  "max_abs_err_over_max_abs_y": float(np.abs(yg - yo).max() / ymax), "tolerance": 1e-12}

    if world > 1 or args.submesh_check:
        nchk, worst, bitw = submesh_parity(cfg, op, y, rank, dev)
        if nchk:
            tt = torch.tensor([worst, 0.0 if bitw else 1.0, float(nchk)], dtype=torch.float64, device=red_dev)
            if world > 1:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            sub = {"vs": "single-rank GPU operator on the 3x3x3-cell sub-box around sampled cells (one next to "
                         "every partition face per rank; partition invariance, SURVEY 8(e))",
                   "cells_per_rank": nchk, "max_abs_err_over_max_abs_y": float(tt[0]),
                   "bitwise": bool(tt[1] == 0.0), "tolerance": 1e-12}
            if parity is None:
                parity = sub
            else:
                parity["partition_invariance"] = sub

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
               "scaling": "strong" if cfg.name.startswith("C5-strong") else "weak",
               "vs_baseline": vs_baseline(cfg, value), "dtype": "f64",
               "data": "synthetic (seeded counter-based uniform[-1,1] z, C-13)",
               "config": workload_desc(cfg, world),
               "gflops_model": per_dof * value / 1e9,
               "roofline": roof, "cpu_baseline": cpu, "parity": parity, "e2e": e2e, "clocks": clk,
               "step_ms": {"mean": ms_per_step, "min": min(step_ms) if step_ms else None,
                           "median": float(np.median(step_ms)) if step_ms else None},
               "gpu_launches": args.steps * info["launches_per_apply"],
               "kernel_info": info,
               "shared_gpu": shared or None,
               "comm": {"transport": transport, "nranks": comm_ranks, "note": halo_note,
                        "halo": "face traces, 2 n^2 doubles per partition-face cell (%d B per cell at k=%d)"
                                % (16 * (cfg.k + 1) ** 2, cfg.k) if world > 1 else None}}
        if timeline is not None:
            out["overlap_timeline"] = timeline
        if world > 1:   # the exchange's cost = t(apply) - t(apply with the halo exchange skipped)
            out["halo_ablation"] = {"ms_per_apply": t / args.steps * 1e3,
                                    "ms_per_apply_no_exchange": tk / args.steps * 1e3,
                                    "what": "same applies with DG_HALO_EXTERNAL (no trace pack, no exchange; "
                                            "stale receive buffers, timing only)"}
        print(json.dumps(out), flush=True)
    op.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def spawn_ranks(n):
    """`python bench.py --gpus N` without torchrun: launch the N ranks (one process per GPU)
    through torch.distributed.run on this node, exactly as the driver does, and return its code."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default=None,
                    help="default: C3 (N=1) / C5 weak, 128x128x64 cells per GPU (N>1); also c1, c2, c3weak, c4-kK, c5weak, c5strong, "
                         "a-kK (the paper's Problem A: periodic, per-cell tensor D, ~4e8 DOFs), "
                         "tg-kK (the Taylor-Green transport operator: b(x) at every point, q = 2p+4)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU-baseline sample budget")
    ap.add_argument("--ref-seconds", type=float, default=120.0, help="reference arm total budget")
    ap.add_argument("--submesh-check", action="store_true", help="partition-invariance check also at N = 1")
    ap.add_argument("--halo", choices=["p2p", "nccl"], default="p2p",
                    help="N > 1: the fused halo (the trace pack stores into the neighbours' buffers over "
                         "NVLink through CUDA IPC; default) or NCCL send/recv from send buffers")
    ap.add_argument("--share-gpu", action="store_true",
                    help="development: N ranks on the visible GPU(s) (gloo + the IPC halo, no NCCL), to "
                         "exercise the N-rank path on a one-GPU box; not a scaling measurement")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
