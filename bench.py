#!/usr/bin/env python
"""Benchmark: FP64 SIPDG Jacobi-PCG iterations on B200 (BASELINE.json metric / config C2).

A "step" is one pass of the whole hot path: one Jacobi-PCG
iteration = pass A (direction update p = D^-1 r + beta p, deferred x update, Ax on the
FP64 tensor cores, p.Ap) + pass B (r -= alpha Ap, r.z, r.r) + device-side scalar control.
value = DOFs x steps / device time  [GDOF/s]  (DOF-iterations per second, all ranks).

  python bench.py                      # N=1 GPU, C2: N=4, 199,712 triangles
  torchrun --nproc-per-node 8 bench.py --gpus 8     # weak scaling, one C2-size tile per rank
  python bench.py --impl reference     # the CPU oracle (the reference arm), same metric/config
  python bench.py --sweep              # degree sweep N=1..8 on C3 (Ax only), JSON lines

Timing: W untimed warm-up steps; K steps bracketed by barrier + synchronize, timed with CUDA
events on the launching stream, max over ranks.  The pass-A+B working set (six K x Np
vectors = 144 MB at C2) exceeds the 126 MB L2, so no flush is needed between steps; the
Ax-only figure rotates through buffers totalling > 4x L2.
"""
import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP64 IPDG Ax GDOF/s and % of HBM roofline vs N; PCG solves/s at 1/2/4/8 B200"
UNIT = "GDOF/s"
C2 = dict(N=4, nx=316, jitter=0.2, diag="random", order="morton", seed=2)


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


KERNEL_NAMES = {1: "k_sipdg", 2: "k_grad+k_flux", 4: "k_pipe", 5: "k_gather", 6: "k_tpb"}
FP64_PEAK_TFLOPS = 36.8  # measured DFMA / DMMA peak on this pool's B200 (profiles/r01_micro_fp64.jsonl)


# ---------------------------------------------------------------- clocks during the timed region
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock"}

    def __init__(self, device):
        self.samples, self.reasons, self.ok = [], 0, False
        self.stop_evt = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self.stop_evt.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.reasons |= int(r)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop_evt.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0}
        s = sorted(self.samples)
        names = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(s)}


# ---------------------------------------------------------------- distributed plumbing
def free_port():
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def self_launch(args):
    """`python bench.py --gpus N` outside torchrun: re-exec this script under torch.distributed.run with N
    ranks on this node (one process per GPU, rendezvous on 127.0.0.1).  Under torchrun the world size
    must equal --gpus."""
    world = int(os.environ.get("WORLD_SIZE", "0") or 0)
    if world:
        if world != args.gpus:
            raise SystemExit("bench.py: WORLD_SIZE=%d but --gpus %d" % (world, args.gpus))
        return
    if args.gpus <= 1:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def dist_setup(backend):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return world, rank, local


def max_over_ranks(v, world, device=None):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def sum_over_ranks(v, world, device=None):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v)], dtype=torch.float64, device=device)
    dist.all_reduce(t)
    return t.item()


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ---------------------------------------------------------------- workload
CONFIGS = {
    # BASELINE.json configs[1]: single-B200 Ax throughput, N=4, ~200k-triangle unstructured square
    "C2": dict(N=4, desc="jittered %dx%d-cell unit square (Morton order, all Dirichlet)" % (C2["nx"], C2["nx"])),
    # configs[3]: Jacobi-PCG pressure Poisson at N=6 on a channel-with-cylinder mesh (~2M triangles), strong scaling
    "C4": dict(N=6, desc="channel [-16,25]x[-22,22] minus the unit square cylinder, graded, 1.84M triangles "
                        "(outflow Dirichlet, other boundaries Neumann)"),
    # configs[4]: weak scaling at N=8, 4M triangles per GPU
    "C5": dict(N=8, desc="one 1414x1414-cell tile (3,998,792 triangles) per GPU, all Dirichlet"),
}


def build_mesh(config, world, rank):
    """Global mesh and element -> rank map (None on one GPU)."""
    from paper_1801_00246_b200 import meshgen
    if config == "C4":
        m = meshgen.cylinder()
        part = None if world == 1 else meshgen.rcb_partition(m["VX"], m["VY"], m["EToV"], world)
        return m, part
    if config == "C5" or world > 1:
        n = 1414 if config == "C5" else C2["nx"]
        px = {1: 1, 2: 2, 4: 2, 8: 4}.get(world, world)
        py = world // px
        mesh, part = meshgen.tiles(n, px, py, jitter=C2["jitter"], seed=C2["seed"])
        return mesh, (part if world > 1 else None)
    m = meshgen.square(C2["nx"], jitter=C2["jitter"], diag=C2["diag"], order=C2["order"], seed=C2["seed"])
    return m, None


def pass_a_bytes_per_elem(Np, precond):
    # reads z = D^-1 r (written by pass B), p_{k-1}, x; writes p_k, x, Ap (8 B each per DOF)
    # + 4 geometric doubles + 8 B neighbour slots.  (Pass B: reads r, Ap, D^-1; writes r, z.)
    vec = 6 * 8 * Np
    return vec + 32 + 8


def ax_flops_per_elem(N):
    Np, Nfp = (N + 1) * (N + 2) // 2, N + 1
    return 8 * Np * Np + 6 * Np * Nfp + 6 * Nfp * Nfp + 18 * Np + 36 * Nfp  # F_min


def traffic_from_profile(N, K, kernel):
    """dram bytes per launch of pass A from the committed ncu capture (profiles/), or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        e = d["pass_a"]
        if e.get("N") == N and e.get("K") == K and e.get("kernel", "k_sipdg") == kernel:
            return e["dram_bytes_per_launch"]
    except Exception:
        pass
    return None


def cpu_oracle_sample(N, iters, nx):
    """Oracle Jacobi-PCG on a bounded sub-mesh of the C2 recipe: returns (GDOF/s, cores, desc, seconds)."""
    import numpy as np
    from oracle import solvers
    from oracle.assemble import assemble
    from oracle.mfree import MFree
    from oracle.refelem import RefElem
    from paper_1801_00246_b200 import meshgen
    m = meshgen.square(nx, jitter=C2["jitter"], diag=C2["diag"], order=C2["order"], seed=C2["seed"])
    ref = RefElem(N)
    mf = MFree(m["VX"], m["VY"], m["EToV"], m["bc"], ref)
    A = assemble(m["VX"], m["VY"], m["EToV"], m["bc"], ref)
    dinv = 1.0 / A.diagonal()
    b = solvers.rhs_mass_interp(m["VX"], m["VY"], m["EToV"], ref, meshgen.sin_sin_forcing).ravel()
    apply = lambda v: mf.apply(v).ravel()  # noqa: E731
    solvers.pcg(apply, b, 0.0, 1, dinv=dinv)  # warm
    t0 = time.perf_counter()
    _, st = solvers.pcg(apply, b, 0.0, iters, dinv=dinv)
    dt = time.perf_counter() - t0
    K = m["EToV"].shape[0]
    try:
        from threadpoolctl import threadpool_info
        blas = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        blas = 1
    desc = ("oracle.solvers.pcg + oracle.mfree (numpy; BLAS threads=%d, elementwise single-threaded) on a "
            "%dx%d-cell C2-recipe sub-mesh (K=%d, N=%d), %d Jacobi-PCG iterations" % (blas, nx, nx, K, N, st["iterations"]))
    return K * ref.Np * st["iterations"] / dt / 1e9, blas, desc, dt


# ---------------------------------------------------------------- our arm
def _solve(op, b, xs, stream, world, dev, precond=1):
    import torch
    torch.cuda.synchronize()
    barrier(world)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    _, sst = op.pcg_solve(b, xs, precond=precond, tol=1e-8, maxit=_solve.maxit)
    s1.record(stream)
    torch.cuda.synchronize()
    return max_over_ranks(s0.elapsed_time(s1), world, dev), sst


_solve.maxit = 100000


def run_ours(args):
    _solve.maxit = args.maxit
    import torch
    from paper_1801_00246_b200 import Ipdg, meshgen
    world, rank, local = dist_setup("nccl")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    N = CONFIGS[args.config]["N"]
    mesh, part = build_mesh(args.config, world, rank)
    if world > 1:
        op = Ipdg.distributed(N, mesh, part, rank, world, device=local)
    else:
        op = Ipdg(N, mesh, device=local)
    if args.variant:
        op.set_variant(args.variant)
    K, Np = op.K, op.Np
    # right-hand side b = J M f_I of the manufactured problem (setup, not timed)
    x_nodes, y_nodes = op.nodes()
    if args.config == "C4":  # f = exp(-((x-2)^2 + y^2)/4)
        f = torch.exp(-((x_nodes - 2.0) ** 2 + y_nodes ** 2) / 4.0)
    else:  # -Lap of sin(pi x / Px) sin(pi y / Py) on the (tiled) domain; Px = Py = 1 on one GPU
        Px = float(mesh["VX"].max() - mesh["VX"].min())
        Py = float(mesh["VY"].max() - mesh["VY"].min())
        f = math.pi ** 2 * (1 / Px ** 2 + 1 / Py ** 2) * torch.sin(math.pi * x_nodes / Px) * torch.sin(math.pi * y_nodes / Py)
    b = op.mass(f)
    x = torch.zeros_like(b)
    stream = torch.cuda.current_stream()
    op.pcg_begin(b, x, precond=1, tol=0.0)
    op.pcg_iterate(args.warmup)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = op.launch_count()
    with ClockSampler(local) as clk:
        e0.record(stream)
        op.pcg_iterate(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
    launches = op.launch_count() - l0
    ms_local = e0.elapsed_time(e1)
    barrier(world)
    ms = max_over_ranks(ms_local, world, dev)
    dofs_total = sum_over_ranks(K * Np, world, dev)
    value = dofs_total * args.steps / (ms / 1e3) / 1e9
    # live per-kernel durations of the dominant kernel (pass A) on the launching stream
    nprof = min(200, max(20, args.steps // 10))
    ms_a, ms_b = op.pcg_iterate_profiled(nprof)
    st = op.pcg_end()
    expected = args.warmup + args.steps + nprof
    if st["iterations"] != expected:
        raise RuntimeError("PCG stopped early (%s) - the timed window would not be %d full iterations" % (st, args.steps))
    avg_a = ms_a / nprof
    pk = peaks()
    bytes_a = pass_a_bytes_per_elem(Np, True) * K
    achieved = bytes_a / (avg_a / 1e3) / 1e9
    flops_a = (ax_flops_per_elem(N) + 6 * Np) * K
    share_a = ms_a / (ms_a + ms_b)
    # Ax alone (rotating buffers > 4x L2), GDOF/s
    nbuf = max(2, int(math.ceil(4 * 126e6 / (2 * 8 * K * Np))))
    us = [torch.rand(K, Np, dtype=torch.float64, device=dev) for _ in range(nbuf)]
    outs = [torch.empty_like(us[0]) for _ in range(nbuf)]
    for i in range(3):
        op.ax(us[i % nbuf], outs[i % nbuf])
    torch.cuda.synchronize()
    nax = 200
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    for i in range(nax):
        op.ax(us[i % nbuf], outs[i % nbuf])
    a1.record(stream)
    torch.cuda.synchronize()
    ax_ms = a0.elapsed_time(a1) / nax
    ax_ms = max_over_ranks(ax_ms, world, dev)
    ax_gdofs = dofs_total / (ax_ms / 1e3) / 1e9
    del us, outs
    # one full Jacobi-PCG solve to 1e-8 (solves/s)
    solve_ms, sst = float("nan"), {"iterations": None, "rel_residual": None}
    xs = torch.zeros_like(b)
    pmg = None
    if not args.no_solve:
        solve_ms, sst = _solve(op, b, xs, stream, world, dev)
        if world == 1:  # NEXT-3: the same solve with the p-multigrid preconditioner (hierarchy built first)
            op.pcg_solve(b, torch.zeros_like(b), precond=3, tol=1e-8, maxit=1)
            pms, pst = _solve(op, b, torch.zeros_like(b), stream, world, dev, precond=3)
            pmg = {"tol": 1e-8, "iterations": pst["iterations"], "ms": round(pms, 3), "solves_per_s": round(1e3 / pms, 3),
                   "rel_residual": pst["rel_residual"], "levels": [d for d, _ in op.pmg_info()],
                   "note": "IPDG_PRECOND_PMG (DESIGN.md R22-R26); setup (hierarchy, graphs) excluded"}
    # e2e through the public API with host buffers, the call a user makes: ipdg_pcg_solve_host copies b and
    # x0 from pinned host memory, solves to 1e-8 and copies x back.  One untimed call first (the library
    # allocates its per-context staging buffers and captures the iteration graphs once per mesh).
    e2e = None
    if not args.no_e2e:
        bh = b.cpu().pin_memory()
        xh = torch.zeros_like(bh).pin_memory()
        op.pcg_solve_host(bh, xh, precond=1, tol=1e-8, maxit=2)
        xh.zero_()
        torch.cuda.synchronize()
        barrier(world)
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        ste = op.pcg_solve_host(bh, xh, precond=1, tol=1e-8, maxit=args.maxit)
        h1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(h0.elapsed_time(h1), world, dev)
        its = max(1, ste["iterations"])
        e2e = {"value": round(dofs_total * its / (e2e_ms / 1e3) / 1e9, 3), "unit": UNIT,
               "h2d_bytes_per_step": int(2 * 8 * K * Np / its), "d2h_bytes_per_step": int(8 * K * Np / its),
               "iterations": ste["iterations"], "ms": round(e2e_ms, 3),
               "note": "ipdg_pcg_solve_host: H2D of b and x0 (pinned), Jacobi-PCG to 1e-8 (%d iterations), D2H of x, "
                       "one call; value = DOFs x iterations / call time; bytes amortised per iteration" % ste["iterations"]}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, cores, desc, secs = cpu_oracle_sample(N, args.cpu_iters, args.cpu_nx)
        cpu = {"value": round(v, 6), "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc,
               "seconds": round(secs, 2), "host_cpus": len(os.sched_getaffinity(0))}
    info = op.info()
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 6), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "%s: Jacobi-PCG iteration (pass A: p-update + SIPDG Ax + p.Ap; pass B: r-update + r.z, r.r) "
                               "on a %s; %d triangles on this rank, N=%d, manufactured right-hand side"
                               % (args.config, CONFIGS[args.config]["desc"], K, N),
                   "N": N, "K_per_gpu": K, "dofs_total": int(dofs_total), "precond": "jacobi",
                   "l2": "working set 6 x K x Np x 8 B = %.0f MB > 126 MB L2 (no flush needed)" % (6 * 8 * K * Np / 1e6),
                   "parallelism": "element partition, %d rank(s)" % world},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk.get("hbm_gbs"), "unit": "GB/s",
                     "frac": round(achieved / pk.get("hbm_gbs"), 4), "traffic": traffic_from_profile(N, K, KERNEL_NAMES.get(info.get("kernel"))),
                     "kernel": "%s<N=%d, PCG pass A>" % (KERNEL_NAMES.get(info.get("kernel"), "?"), N),
                     "avg_launch_ms": round(avg_a, 5),
                     "algorithmic_bytes_per_launch": bytes_a, "share_of_step": round(share_a, 3),
                     "fp64_tflops": round(flops_a / (avg_a / 1e3) / 1e12, 2),
                     "fp64_frac": round(flops_a / (avg_a / 1e3) / 1e12 / FP64_PEAK_TFLOPS, 4),
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" + (" (fallback)" if pk.get("_fallback") else "")},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "ax_only": {"gdofs": round(ax_gdofs, 3), "ms": round(ax_ms, 5), "buffers_rotated": nbuf},
        "pcg_solve": {"tol": 1e-8, "iterations": sst["iterations"], "ms": (round(solve_ms, 3) if solve_ms == solve_ms else None),
                      "solves_per_s": (round(1e3 / solve_ms, 3) if solve_ms == solve_ms else None), "rel_residual": sst["rel_residual"]},
        "pcg_solve_pmg": pmg,
        "kernel_config": info,
    }
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# ---------------------------------------------------------------- reference arm: the CPU oracle
def run_reference(args):
    world, rank, local = dist_setup("gloo")
    if rank != 0:
        return
    N = C2["N"]
    # each step: one oracle Jacobi-PCG iteration on a bounded C2-recipe sub-mesh
    import numpy as np
    from oracle import solvers
    from oracle.assemble import assemble
    from oracle.mfree import MFree
    from oracle.refelem import RefElem
    from paper_1801_00246_b200 import meshgen
    nx = args.ref_nx
    m = meshgen.square(nx, jitter=C2["jitter"], diag=C2["diag"], order=C2["order"], seed=C2["seed"])
    ref = RefElem(N)
    mf = MFree(m["VX"], m["VY"], m["EToV"], m["bc"], ref)
    A = assemble(m["VX"], m["VY"], m["EToV"], m["bc"], ref)
    dinv = 1.0 / A.diagonal()
    b = solvers.rhs_mass_interp(m["VX"], m["VY"], m["EToV"], ref, meshgen.sin_sin_forcing).ravel()
    apply = lambda v: mf.apply(v).ravel()  # noqa: E731
    solvers.pcg(apply, b, 0.0, args.warmup, dinv=dinv)
    t0 = time.perf_counter()
    _, st = solvers.pcg(apply, b, 0.0, args.steps, dinv=dinv)
    dt = time.perf_counter() - t0
    K = m["EToV"].shape[0]
    value = K * ref.Np * st["iterations"] / dt / 1e9
    try:
        from threadpoolctl import threadpool_info
        blas = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        blas = 1
    desc = ("oracle.solvers.pcg + oracle.mfree on a %dx%d-cell C2-recipe sub-mesh (K=%d, N=%d); each step one "
            "Jacobi-PCG iteration; BLAS threads=%d" % (nx, nx, K, N, blas))
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3 / max(1, st["iterations"]), 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C2 recipe (bounded CPU sample, see cpu_baseline.sample)", "N": N},
            "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": blas, "kind": "oracle", "sample": desc},
            "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ---------------------------------------------------------------- NEXT rows, measured on C2
def run_next(args):
    """NEXT-1: screened Poisson -L + lambda with the block-Jacobi scaled inverse mass vs point
    Jacobi -- iterations to 1e-8, device time per iteration, solves/s.  NEXT-2: DG gradient / divergence
    (Eqs. INS_SD_4_1/4_2) -- time per call and GB/s on algorithmic bytes (read 1 or 2 fields, write 2 or 1,
    + 48 B of geometry/connectivity per element)."""
    import torch
    from paper_1801_00246_b200 import Ipdg, meshgen
    pk = peaks()
    mesh = meshgen.square(C2["nx"], jitter=C2["jitter"], diag=C2["diag"], order=C2["order"], seed=C2["seed"])
    stream = torch.cuda.current_stream()
    for N in (4, 8):
        op = Ipdg(N, mesh)
        K, Np = op.K, op.Np
        x_nodes, y_nodes = op.nodes()
        f = math.pi ** 2 * 2 * torch.sin(math.pi * x_nodes) * torch.sin(math.pi * y_nodes)
        rhs = {"smooth sin(pi x) sin(pi y)": op.mass(f),
               "random U(-1,1)": op.mass(torch.from_numpy(meshgen.uniform_field(K, Np, seed=77)).cuda())}
        for (rname, b), lam, pc in [(r, l, q) for r in rhs.items() for l in (1e5, 1e3) for q in (2, 1)]:
            if True:
                op.pcg_solve(b, torch.zeros_like(b), lam=lam, precond=pc, tol=1e-8, maxit=2)  # setup, graphs
                x = torch.zeros_like(b)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                _, st = op.pcg_solve(b, x, lam=lam, precond=pc, tol=1e-8, maxit=20000)
                e1.record(stream)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1)
                x = torch.zeros_like(b)
                op.pcg_begin(b, x, lam=lam, precond=pc, tol=0.0)
                op.pcg_iterate_profiled(3)
                ma, mb = op.pcg_iterate_profiled(50)
                op.pcg_end()
                print(json.dumps({"next": "NEXT-1 screened Poisson PCG", "config": "C2 mesh", "N": N, "K": K, "lambda": lam, "rhs": rname,
                                  "precond": {1: "jacobi", 2: "block-jacobi (scaled inverse mass)"}[pc],
                                  "iterations": st["iterations"], "rel_residual": st["rel_residual"], "solve_ms": round(ms, 3),
                                  "solves_per_s": round(1e3 / ms, 2), "pass_a_us": round(1e3 * ma / 50, 2),
                                  "pass_b_us": round(1e3 * mb / 50, 2)}), flush=True)
        p = torch.rand(K, Np, dtype=torch.float64, device="cuda")
        uy = torch.rand_like(p)
        for name, fn, nin, nout in (("G p", lambda: op.dg_grad(p), 1, 2), ("D u", lambda: op.dg_div(p, uy), 2, 1)):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(50):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 50
            byt = (8 * Np * (nin + nout) + 48) * K
            print(json.dumps({"next": "NEXT-2 DG %s (central fluxes)" % name, "config": "C2 mesh", "N": N, "K": K,
                              "us": round(1e3 * ms, 2), "gdofs": round(K * Np / (ms / 1e3) / 1e9, 2),
                              "hbm_gbs_algorithmic": round(byt / (ms / 1e3) / 1e9, 1),
                              "hbm_frac": round(byt / (ms / 1e3) / 1e9 / pk["hbm_gbs"], 4)}), flush=True)
        # NEXT-3: p-multigrid V-cycle (one application) and NEXT-4: subcycling advection operator
        r = torch.rand(K, Np, dtype=torch.float64, device="cuda")
        op.pmg_apply(r)
        nq = (3 * N + 2) // 2 + 1
        nc, ncf, nfp = nq * nq, nq, N + 1
        adv_flop = 2 * (4 * nc * Np + 8 * nc * Np + 3 * ncf * nfp * 8 + 2 * Np * 3 * ncf)  # per element (MACs x 2)
        fl = [torch.rand(K, Np, dtype=torch.float64, device="cuda") for _ in range(4)]
        for name, fn in (("NEXT-3 p-multigrid V-cycle", lambda: op.pmg_apply(r)),
                         ("NEXT-4 subcycling advection N~(U_bar, U~)", lambda: op.advect(*fl))):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(20):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 20
            line = {"next": name, "config": "C2 mesh", "N": N, "K": K, "us": round(1e3 * ms, 2),
                    "gdofs": round(K * Np / (ms / 1e3) / 1e9, 2)}
            if name.startswith("NEXT-4"):
                byt = (8 * Np * 6 + 48) * K
                line.update({"fp64_tflops": round(adv_flop * K / (ms / 1e3) / 1e12, 2),
                             "fp64_frac": round(adv_flop * K / (ms / 1e3) / 1e12 / FP64_PEAK_TFLOPS, 4),
                             "hbm_gbs_algorithmic": round(byt / (ms / 1e3) / 1e9, 1), "bound": "fp64",
                             "flop_per_elem": adv_flop})
            else:
                line["levels"] = [[d, round(l, 4)] for d, l in op.pmg_info()]
            print(json.dumps(line), flush=True)
        del op
        torch.cuda.empty_cache()


# ---------------------------------------------------------------- degree sweep (C3), Ax only
def run_sweep(args):
    import torch
    from paper_1801_00246_b200 import Ipdg, meshgen
    pk = peaks()
    nx = args.sweep_nx
    mesh = meshgen.square(nx, jitter=0.2, diag="random", order="morton", seed=3)
    stream = torch.cuda.current_stream()
    for N, variant in [(N, v) for N in range(1, 9) for v in args.sweep_variants if v != 5 or N <= 4]:
        op = Ipdg(N, mesh)
        op.set_variant(variant)
        K, Np = op.K, op.Np
        nbuf = max(2, int(math.ceil(4 * 126e6 / (2 * 8 * K * Np))))
        us = [torch.rand(K, Np, dtype=torch.float64, device="cuda") for _ in range(nbuf)]
        outs = [torch.empty_like(us[0]) for _ in range(nbuf)]
        for i in range(3):
            op.ax(us[i % nbuf], outs[i % nbuf])
        torch.cuda.synchronize()
        n = 50
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(n):
            op.ax(us[i % nbuf], outs[i % nbuf])
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        bmin = (16 * Np + 48) * K
        fmin = ax_flops_per_elem(N) * K
        t_roof = max(bmin / (pk["hbm_gbs"] * 1e9), fmin / (FP64_PEAK_TFLOPS * 1e12))
        print(json.dumps({"sweep": "C3", "N": N, "variant": variant, "K": K, "dofs": K * Np, "ms": round(ms, 5),
                          "gdofs": round(K * Np / (ms / 1e3) / 1e9, 3),
                          "hbm_gbs_algorithmic": round(bmin / (ms / 1e3) / 1e9, 1),
                          "hbm_frac": round(bmin / (ms / 1e3) / 1e9 / pk["hbm_gbs"], 4),
                          "fp64_tflops": round(fmin / (ms / 1e3) / 1e12, 2),
                          "method_roofline_frac": round(t_roof / (ms / 1e3), 4),
                          "bound": "hbm" if bmin / (pk["hbm_gbs"] * 1e9) > fmin / (FP64_PEAK_TFLOPS * 1e12) else "fp64",
                          "kernel_config": op.info()}), flush=True)
        del us, outs, op
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--maxit", type=int, default=100000, help="iteration cap of the timed full solve")
    ap.add_argument("--cpu-iters", type=int, default=600)
    ap.add_argument("--cpu-nx", type=int, default=100)
    ap.add_argument("--ref-nx", type=int, default=50)
    ap.add_argument("--variant", type=int, default=0, help="operator kernel variant (0 auto)")
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--next", action="store_true", help="NEXT-1 / NEXT-2 measurements (SURVEY 8.6) on the C2 mesh")
    ap.add_argument("--sweep-nx", type=int, default=707)
    ap.add_argument("--sweep-variants", type=int, nargs="+", default=[0], help="0 auto, 1 fused, 2 split, 4 pipelined fused, 5 gather (N<=4)")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    self_launch(args)
    if args.impl == "reference":
        run_reference(args)
    elif args.sweep:
        run_sweep(args)
    elif args.next:
        run_next(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
