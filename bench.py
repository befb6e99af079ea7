#!/usr/bin/env python
"""Benchmark: Gray–Scott cell-updates/s per RK step (fp64) on 1..8 B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Headline workload (BASELINE configs[4], weak scaling): a 3D
Gray–Scott z-slab of 512^3 cells per GPU (global 512 x 512 x 512N, h = 2.5/64, one seeded
cube per 512^3 block), integrated with Dormand–Prince 5(4) under error control
(atol = rtol = 1e-6, dt0 = 1): one "step" = one accepted adaptive step, i.e. the whole hot
path: stage values, halo exchange, stencil RHS, final combination, embedded error, max
norm + allreduce, host controller.  value = cells x accepted steps
/ device time (max over ranks).  RK4 fixed-step is measured in the same run ("extra").

Timing: W warm-up steps, then K steps between barrier + synchronize, CUDA events on the
library's stream (torch's current stream).  Arrays are 2 GiB >> 126 MB L2, so no flush is
needed.  Roofline: the fused stage kernel (K3), algorithmic bytes counted by the library
per launch (rk_stats.stage_bytes) over its CUDA-event-timed launch durations.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_PER_GPU = 512
TOL = 1e-6
H = 2.5 / 64  # DESIGN.md R-4: h fixed at the paper's 64^3 spacing


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """dram bytes per launch of the stage kernel from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return None


class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.result = None
        if not self.proc:
            return
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if sm:
            self.result = {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx,
                           "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------------------
# reference arm / CPU baseline: the oracle (test infrastructure) on the host cores
# ---------------------------------------------------------------------------------------
def oracle_try_seconds(nz_sample: int, scheme_name: str = "dopri5"):
    import oracle
    import rk_inputs
    n = N_PER_GPU
    u0 = rk_inputs.gray_scott_ic(n, n, nz_sample, seed=42)
    p = oracle.gray_scott_problem(n, n, nz_sample, h=H)
    t = time.perf_counter()
    if scheme_name == "dopri5":
        un, err = oracle.step(p, oracle.DOPRI5, 0.0, 1.0, u0, with_error=True)
        k1 = oracle.rhs(p, u0)
        E = oracle.error_ratio_max(err, u0, k1, 1.0, TOL, TOL)
        oracle.controller(E, 1.0)
    else:
        oracle.step(p, oracle.RK4, 0.0, 1.0, u0)
    return time.perf_counter() - t, n * n * nz_sample


def _oracle_worker(args):
    """One host core: the unmodified single-threaded oracle on its own slab (built before the
    barrier, so only the DOPRI5 tries are timed).  Returns (start, end, cells) wall times."""
    nz_sample, tries, barrier = args
    import oracle
    import rk_inputs
    n = N_PER_GPU
    u0 = rk_inputs.gray_scott_ic(n, n, nz_sample, seed=42)
    p = oracle.gray_scott_problem(n, n, nz_sample, h=H)
    oracle.lib()
    barrier.wait()
    t0 = time.time()
    for _ in range(tries):
        un, err = oracle.step(p, oracle.DOPRI5, 0.0, 1.0, u0, with_error=True)
        E = oracle.error_ratio_max(err, u0, oracle.rhs(p, u0), 1.0, TOL, TOL)
        oracle.controller(E, 1.0)
    return t0, time.time(), n * n * nz_sample * tries


def oracle_all_cores(nz_each=4, tries=4):
    """The oracle on the box's host cores: W independent single-threaded oracle processes (the
    oracle itself is never modified or threaded), each running DOPRI5 tries on its own
    512x512xnz_each slab; throughput = all cells / (last end - first start).  W is capped at 64
    so the oracle's textbook storage (every k_j, ~0.25 GB per 1M cells) stays under ~17 GB."""
    import multiprocessing as mp
    workers = max(1, min(os.cpu_count() or 1, 64))
    ctx = mp.get_context("spawn")  # the parent may hold a CUDA context: never fork it
    with ctx.Manager() as m:
        bar = m.Barrier(workers)
        with ctx.Pool(workers) as pool:
            res = pool.map(_oracle_worker, [(nz_each, tries, bar)] * workers)
    t0 = min(r[0] for r in res)
    t1 = max(r[1] for r in res)
    cells = sum(r[2] for r in res)
    return cells / (t1 - t0), workers, t1 - t0


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_small_configs():
    """the oracle on BASELINE configs[0..2] in full, one host core (the GPU side of
    the same runs is extra.small_configs / extra.exp512)."""
    import oracle
    import rk_inputs
    out = {}
    n1 = 100000  # configs[0]: du/dt = -u, RK4, t in [0, 1], dt = 0.1
    t = time.perf_counter()
    _, steps = oracle.integrate_const(oracle.exp_problem(n1, -1.0), oracle.RK4, rk_inputs.exp_decay_u0(n1),
                                      0.0, 1.0, 0.1)
    sec = time.perf_counter() - t
    out["config0_exp_rk4"] = {"value": n1 * steps / sec, "unit": "element-updates/s", "seconds": sec, "steps": steps}
    n2 = 1000000  # configs[1]: logistic, DOPRI5 adaptive tol 1e-8 on [-5, 5]
    t = time.perf_counter()
    _, acc, rej, _ = oracle.integrate_adaptive(oracle.logistic_problem(n2), oracle.DOPRI5, rk_inputs.logistic_u0(n2),
                                               -5.0, 5.0, 0.1, 1e-8, 1e-8)
    sec = time.perf_counter() - t
    out["config1_logistic_dopri5"] = {"value": n2 * (acc + rej) / sec, "unit": "element-tries/s", "seconds": sec,
                                      "accepted": acc, "rejected": rej}
    n3 = 64  # configs[2]: Gray-Scott 64^3, RK4 dt = 1, t in [0, 20]
    u0 = rk_inputs.gray_scott_ic(n3, n3, n3, seed=42)
    t = time.perf_counter()
    _, steps = oracle.integrate_const(oracle.gray_scott_problem(n3, n3, n3), oracle.RK4, u0, 0.0, 20.0, 1.0)
    sec = time.perf_counter() - t
    out["config2_gs64_rk4"] = {"value": n3 ** 3 * steps / sec, "unit": "cell-updates/s", "seconds": sec, "steps": steps}
    return out


def oracle_full_512():
    """SURVEY §8d oracle plan at full size (opt-in leg cpu_full, ~1 min, ~25 GB of host RAM): the
    unmodified single-threaded oracle on the whole 512^3 configs[3] grid -- 2 RK4 steps (dt = 1)
    and 1 DOPRI5 error-controlled try (7 RHS evaluations, error ratio, max norm, controller)."""
    import oracle
    import rk_inputs
    n = N_PER_GPU
    u0 = rk_inputs.gray_scott_ic(n, n, n, seed=42)
    p = oracle.gray_scott_problem(n, n, n, h=H)
    oracle.lib()
    t = time.perf_counter()
    u1 = oracle.step(p, oracle.RK4, 0.0, 1.0, u0)
    oracle.step(p, oracle.RK4, 1.0, 1.0, u1)
    t_rk4 = time.perf_counter() - t
    del u1
    t = time.perf_counter()
    un, err = oracle.step(p, oracle.DOPRI5, 0.0, 1.0, u0, with_error=True)
    E = oracle.error_ratio_max(err, u0, oracle.rhs(p, u0), 1.0, TOL, TOL)
    acc, dtn = oracle.controller(E, 1.0)
    t_dp = time.perf_counter() - t
    cells = n ** 3
    return {"rk4": {"value": 2 * cells / t_rk4, "unit": "cell-updates/s", "seconds": t_rk4, "steps": 2},
            "dopri5_try": {"value": cells / t_dp, "unit": "cell-tries/s", "seconds": t_dp, "E": E,
                           "accepted": bool(acc)},
            "cores": 1, "cpu_model": cpu_model(),
            "sample": "the whole 512^3 grid (configs[3]), single-threaded C oracle (-O2 -ffp-contract=off)"}


def cpu_baseline(nz_sample=128):
    secs, cells = oracle_try_seconds(nz_sample)
    single = cells / secs
    try:
        v, workers, wall = oracle_all_cores()
    except Exception as e:  # report the single-core number rather than nothing
        return {"value": single, "unit": "cell-updates/s", "cores": 1, "kind": "oracle",
                "sample": f"one DOPRI5 try on a 512x512x{nz_sample} slab, single thread, {secs:.1f} s "
                          f"(all-core run failed: {e})"}
    try:
        small = oracle_small_configs()
    except Exception as e:
        small = {"error": str(e)}
    return {"value": v, "unit": "cell-updates/s", "cores": workers, "kind": "oracle",
            "single_core_value": single, "cpu_model": cpu_model(), "small_configs_single_core": small,
            "sample": f"all host cores: {workers} processes of the single-threaded C oracle (-O2 "
                      f"-ffp-contract=off), each 4 DOPRI5 error-controlled tries (7 RHS evals, "
                      f"error ratio, max norm, controller) on its own 512x512x4 periodic slab, "
                      f"{wall:.1f} s wall; single core on a 512x512x{nz_sample} slab: "
                      f"{single:.3g} cell-updates/s ({secs:.1f} s)"}


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    oracle_all_cores(tries=1)  # warm-up: page in the library and numpy in every worker
    tot, cells, workers = 0.0, 0, 1
    for _ in range(args.steps):
        v, workers, wall = oracle_all_cores()
        tot += wall
        cells += v * wall
    v = cells / tot
    line = {"impl": "reference", "metric": "gray_scott_cell_updates_per_s", "value": v,
            "unit": "cell-updates/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Gray-Scott IC, DESIGN.md R-6)",
            "config": {"workload": "gray_scott_dopri5_adaptive_512^3_per_gpu",
                       "sample": f"per step: {workers} oracle processes x 4 DOPRI5 tries on "
                                 f"512x512x4 slabs"},
            "cpu_baseline": {"value": v, "unit": "cell-updates/s", "cores": workers, "kind": "oracle",
                             "sample": f"each step = {workers} single-threaded oracle processes, "
                                       f"4 DOPRI5 tries each on its own 512x512x4 slab"},
            "e2e": {"value": v, "unit": "cell-updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------
# B/cell per step of each scheme's fused stage-by-stage schedule (the gate's
# bytes; this build moves fewer for DOPRI5 / CK54 through the write-ahead stage)
SURVEY_BYTES = {"euler": 32, "rk4": 208, "cash_karp54": 432, "dopri5": 432}
# K6 / K8 roofline: algorithmic fp64 (non-FMA) operations per cell-step
K6_OPS = {"rk4": 168, "midpoint": 78, "modified_midpoint": 125}
K8_LAUNCHES = {"rk4": 2, "midpoint": 1, "modified_midpoint": 2}  # K8 launches per step (Gragg: pair + K3 last stage)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_PER_GPU, help="cells per axis per GPU (x, y, z-slab)")
    ap.add_argument("--legs", default="adaptive,rk4,rk4_k3,repeats,try_loop,device_loop,halo,exposed,strong,strong_emul,rk4_native,rk4_k6,exp512,small,e2e,cpu",
                    help="comma list of legs (profiling runs use e.g. --legs rk4)")
    ap.add_argument("--no-extra", action="store_true", help="same as --legs adaptive")
    ap.add_argument("--overlap", type=int, default=1, help="halo exchange overlapped (N > 1)")
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference" or os.environ.get("BENCH_ALLOW_SHORT")
    legs = set(args.legs.split(","))
    if args.no_extra:
        legs = {"adaptive"}

    rank, world, local = dist_setup()
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    import paper_2309_05331_b200 as rk
    import rk_inputs

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    if world > 1:
        ctx = rk.Context.from_torch_distributed(local, stream)
    else:
        ctx = rk.Context(0, 1, local, stream)

    n = args.n
    nzg = n * world
    st = ctx.grid(n, n, nzg, 2)
    st.set_rhs_gray_scott(h=H)
    st.set_option(rk.OPT_HALO_OVERLAP, args.overlap)
    u0 = rk_inputs.gray_scott_ic(n, n, nzg, seed=42, z0=st.begin, nzl=st.local, zblocks=world)
    u0_dev = torch.from_numpy(u0).cuda(local)
    st.set(u0_dev)
    cells_local = n * n * st.local
    cells_total = n * n * nzg
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    peak, peak_src = peaks()
    traffic = ncu_traffic() or {}

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def survey_gate(bytes_per_cell, cell_tries, ms):
        eff = bytes_per_cell * cell_tries / (ms / 1e3) / 1e9
        return {"bytes_per_cell": bytes_per_cell, "effective_gbs": eff, "frac": eff / peak, "target_frac": 0.70}

    def halo_of(s, p2p=False):
        # halo time (comm-stream CUDA events around each exchange) and its GB/s, reported
        # separately; one GPU: the loopback self-exchange (a device copy)
        if not s["halo_exchanges"]:
            return None
        gbs = (s["halo_bytes"] / (s["halo_ms"] / 1e3) / 1e9) if s["halo_ms"] else None
        return {"exchanges": s["halo_exchanges"], "ms_per_exchange": s["halo_ms"] / s["halo_exchanges"],
                "bytes_per_exchange": s["halo_bytes"] / s["halo_exchanges"],
                "transport": ("p2p stores" if p2p else "nccl") + (" over nvlink" if world > 1 else
                                                                  " (loopback on one GPU)"),
                ("nvlink_gbs" if world > 1 else "gbs"): gbs}

    # ---- headline: DOPRI5 adaptive, one accepted step per "step" ---------------------
    state = {"t": 0.0, "dt": 1.0}

    def adaptive_step():
        tries = 0
        while True:
            acc, E, dtn = st.try_step("dopri5", state["t"], state["dt"], TOL, TOL)
            tries += 1
            if acc:
                state["t"] += state["dt"]
                state["dt"] = dtn
                return tries
            state["dt"] = dtn

    T1 = 20.0  # configs[3]/[4]: DOPRI5 adaptive over t in [0, 20], dt0 = 1

    def integrate_step(src):
        """One bench "step" = one pass of the whole hot path over the configs[3]/[4] input:
        rk_state_set of the seeded IC (src: device tensor, or pinned host tensor for e2e) and
        rk_integrate_adaptive from t = 0 to 20 (the a8 driver: every try's stages, halo path,
        error max + allreduce, controller, FSAL).  Returns (accepted, rejected)."""
        st.set(src)
        return st.integrate_adaptive("dopri5", 0.0, T1, 1.0, TOL, TOL)

    def kernel_traffic(rec, name):
        # ncu DRAM bytes per launch of the kernel `name` in one captured try
        pl = [b for nm, b in rec.get("per_launch", []) if name in nm]
        return sum(pl) / len(pl) if pl else None

    def adaptive_leg():
        for _ in range(args.warmup):
            integrate_step(u0_dev)
        st.reset_stats()
        barrier()
        acc = rej = 0
        with ClockSampler(local) as clk:
            ev0.record(stream)
            for _ in range(args.steps):
                a, r = integrate_step(u0_dev)
                acc, rej = acc + a, rej + r
            ev1.record(stream)
            barrier()
        ms = max_over_ranks(ev0.elapsed_time(ev1))
        s = st.stats()
        # Per-launch durations for the roofline come from a second, identical pass with a CUDA
        # event pair around every stage launch (RK_OPT_TIMING): recording ~280 events per
        # integration costs ~1.4 % of the step time, so the headline pass above runs without them.
        st.reset_stats()
        st.set_option(rk.OPT_TIMING, 1)
        barrier()
        for _ in range(args.steps):
            integrate_step(u0_dev)
        barrier()
        s_t = st.stats()
        st.set_option(rk.OPT_TIMING, 0)
        k_ms = s_t["stage_kernel_ms"] * s["stage_launches"] / max(1, s_t["stage_launches"])
        all_gbs = s["stage_bytes"] / (k_ms / 1e3) / 1e9 if k_ms > 0 else None
        step_bytes = s["stage_bytes"] / max(1, s["tries"])
        # the three kernel roles of a DOPRI5 try on the K8 schedule: K3 stage
        # launches (k1 after a rejection, stage 4, the write-ahead stage 5), the K8 head pair
        # (stages 2 + 3) and the K8 tail pair (stages 6 + 7 + ratio), each from the CUDA-event
        # pass: launches, algorithmic bytes, time
        roles = {
            "k3_stages": ("gs_stage_kernel (K3: fused stage value + 7-pt stencil + reaction + epilogue; "
                          "stage 4, the write-ahead stage 5, k1 after a rejection)",
                          s_t["stage_launches"] - s_t["pair_launches"],
                          s_t["stage_bytes"] - s_t["pair_bytes"],
                          s_t["stage_kernel_ms"] - s_t["pair_kernel_ms"]),
            "k8_head_pair": ("gs_pair_kernel (K8 DOPRI5 head pair: stages 2 + 3, k2 and k3)",
                             s_t["head_launches"], s_t["head_bytes"], s_t["head_kernel_ms"]),
            "k8_tail_pair": ("gs_pair_kernel (K8 DOPRI5 tail pair: stages 6 + 7, u_new, FSAL k7, ratio)",
                             s_t["pair_launches"] - s_t["head_launches"], s_t["pair_bytes"] - s_t["head_bytes"],
                             s_t["pair_kernel_ms"] - s_t["head_kernel_ms"]),
        }
        kern = {}
        for key, (name, nl, nb, nms) in roles.items():
            if nl <= 0 or nms <= 0:
                continue
            g = nb / (nms / 1e3) / 1e9
            kern[key] = {"kernel": name, "launches": nl, "achieved": g, "unit": "GB/s", "frac": g / peak,
                         "algorithmic_bytes_per_launch": nb / nl, "avg_launch_ms": nms / nl,
                         "share_of_stage_time": nms / s_t["stage_kernel_ms"]}
        # the dominant kernel (by function, as ncu lists them): gs_stage_kernel (K3) or
        # gs_pair_kernel (K8 head + tail pairs), whichever holds more of the stage time here
        k3 = roles["k3_stages"]
        k8 = ("gs_pair_kernel (K8 stage pairs: the DOPRI5 head pair, stages 2 + 3, and the tail pair, "
              "stages 6 + 7 + ratio)", s_t["pair_launches"], s_t["pair_bytes"], s_t["pair_kernel_ms"])
        dom, dom_fn = (k8, "gs_pair_kernel") if k8[3] > k3[3] else (k3, "gs_stage_kernel")
        d_name, d_launches, d_bytes, d_ms = dom
        achieved = d_bytes / (d_ms / 1e3) / 1e9 if d_ms > 0 else None
        line = {
            "metric": "gray_scott_cell_updates_per_s",
            # a cell-update = one cell advanced by one ACCEPTED Runge-Kutta step
            "value": cells_total * acc / (ms / 1e3),
            "unit": "cell-updates/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded Gray-Scott IC, DESIGN.md R-6)",
            "config": {"workload": "gray_scott_dopri5_adaptive_512^3_per_gpu", "nx": n, "ny": n,
                       "nz_global": nzg, "nz_per_gpu": int(st.local), "h": H, "atol": TOL,
                       "rtol": TOL, "scheme": "dopri5 (FSAL, error-controlled)",
                       "step": "one rk_integrate_adaptive call over t in [0, 20], dt0 = 1, from the "
                               "seeded IC (rk_state_set from HBM inside the timed region)",
                       "accepted_per_step": acc / args.steps, "rejected_per_step": rej / args.steps,
                       "tries": s["tries"], "ms_per_accepted_rk_step": ms / max(1, acc),
                       "ms_per_try": ms / max(1, s["tries"]),
                       "halo_overlap": bool(args.overlap),
                       "l2": "no flush: every array is 2 GiB per GPU, >> 126 MB L2",
                       "parallelism": f"z-slab x{world} (NCCL send/recv halos + allreduce max)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None,
                         "frac_of_datasheet_8000": (achieved / 8000.0) if achieved else None,
                         "traffic": kernel_traffic(traffic.get("dopri5_adaptive", {}), dom_fn),
                         "traffic_source": "not measured in this run: dram__bytes_read.sum + "
                                           f"dram__bytes_write.sum per {dom_fn} launch of one DOPRI5 try "
                                           "from the committed ncu --set full capture "
                                           f"(profiles/ncu_traffic.json: {str(traffic.get('_source', '?'))[:40]})",
                         "kernel": d_name + f" -- the dominant kernel, {d_ms / s_t['stage_kernel_ms']:.0%} "
                                   "of the stage time; every role is in `kernels`",
                         "algorithmic_bytes_per_launch": d_bytes / max(1, d_launches),
                         "algorithmic_bytes_per_cell_try": step_bytes / cells_local,
                         "avg_launch_ms": d_ms / max(1, d_launches),
                         "launches": d_launches, "peak_source": peak_src,
                         "kernels": kern,
                         "all_stage_launches": {"achieved": all_gbs, "frac": all_gbs / peak if all_gbs else None,
                                                "algorithmic_bytes_per_cell_try": step_bytes / cells_local,
                                                "note": "every stage launch of a try together (K3 + K8)"},
                         "timing": "achieved = algorithmic bytes / CUDA-event durations of the same stage "
                                   "launches in a second pass of the K integrations (per-launch events "
                                   "off in the headline pass)",
                         # SURVEY §8d gate: cells x tries x 528 B (its DOPRI5 adaptive schedule)
                         # over the whole timed region, against >= 0.70 of the measured peak
                         "survey_gate": survey_gate(528, cells_local * s["tries"], ms),
                         # the K8 pairs are issue-bound kernels that move fewer bytes: their own HBM
                         # fraction is low while the try beats the stage-by-stage (K3) schedule's HBM
                         # floor -- 480 B/cell/try at the measured peak -- over the whole timed region
                         "vs_stage_by_stage_floor": {
                             "bytes_per_cell_try": 480,
                             "floor_ms_per_try": 480 * cells_local / (peak * 1e9) * 1e3,
                             "ms_per_try": ms / max(1, s["tries"]),
                             "floor_over_measured": (480 * cells_local / (peak * 1e9) * 1e3)
                                                    / (ms / max(1, s["tries"]))}},
            "gpu_launches": s["kernel_launches"],
            "clocks": getattr(clk, "result", None),
        }
        h = halo_of(s)
        if h:
            line["halo"] = h
        return line

    # the try_step loop of round 1 (one accepted step per "step", Python-driven): kept as an extra
    state = {"t": 0.0, "dt": 1.0}

    def adaptive_step():
        tries = 0
        while True:
            acc, E, dtn = st.try_step("dopri5", state["t"], state["dt"], TOL, TOL)
            tries += 1
            if acc:
                state["t"] += state["dt"]
                state["dt"] = dtn
                return tries
            state["dt"] = dtn

    def try_loop_leg():
        st.set(u0_dev)
        state["t"], state["dt"] = 0.0, 1.0
        for _ in range(args.warmup):
            adaptive_step()
        barrier()
        ev0.record(stream)
        tries = sum(adaptive_step() for _ in range(args.steps))
        ev1.record(stream)
        barrier()
        ms = max_over_ranks(ev0.elapsed_time(ev1))
        return {"value": cells_total * args.steps / (ms / 1e3), "unit": "cell-updates/s",
                "ms_per_step": ms / args.steps, "tries": tries,
                "config": "rk_try_step driven from Python, one accepted DOPRI5 step per step"}

    def rk4_leg(overlap: int, scheme: str = "rk4", p2p: int = 0, loopback: int = 0, k8_ok: bool = True):
        st.set_option(rk.OPT_HALO_OVERLAP, overlap)
        st.set_option(rk.OPT_HALO_LOOPBACK, loopback)
        st.set_option(rk.OPT_HALO_P2P, p2p)
        st.set(u0_dev)
        # Adams–Bashforth k: the first k-1 steps are RKF78 bootstrap steps; keep them untimed
        nwarm = max(args.warmup, int(scheme.lstrip("abm")) if scheme.startswith("ab") else 0)
        for _ in range(nwarm):
            st.do_step(scheme, 0.0, 1.0)
        st.set_option(rk.OPT_TIMING, 1)
        st.reset_stats()
        barrier()
        ev0.record(stream)
        for k in range(args.steps):
            st.do_step(scheme, float(k), 1.0)
        ev1.record(stream)
        barrier()
        ms4 = max_over_ranks(ev0.elapsed_time(ev1))
        s4 = st.stats()
        st.set_option(rk.OPT_TIMING, 0)
        st.set_option(rk.OPT_HALO_OVERLAP, args.overlap)
        st.set_option(rk.OPT_HALO_P2P, 0)
        st.set_option(rk.OPT_HALO_LOOPBACK, 0)
        a4 = s4["stage_bytes"] / (s4["stage_kernel_ms"] / 1e3) / 1e9 if s4["stage_kernel_ms"] else None
        k8 = (k8_ok and world == 1 and not loopback and not p2p and scheme in K8_LAUNCHES
              and s4["stage_launches"] == K8_LAUNCHES[scheme] * args.steps)
        out = {"value": cells_total * args.steps / (ms4 / 1e3), "ms_per_step": ms4 / args.steps,
               "halo_overlap": bool(overlap), "scheme": scheme,
               "halo_path": ("p2p" if p2p else "nccl") + (" (loopback)" if loopback else ""),
               "roofline": {"bound": "hbm", "achieved": a4, "peak": peak, "unit": "GB/s",
                            "frac": a4 / peak if a4 else None,
                            "traffic": traffic.get(scheme, {}).get("bytes_per_launch"),
                            "algorithmic_bytes_per_cell_step": s4["stage_bytes"] / args.steps / cells_local,
                            "avg_launch_ms": s4["stage_kernel_ms"] / max(1, s4["stage_launches"])},
               "gpu_launches": s4["kernel_launches"]}
        if scheme in SURVEY_BYTES:  # SURVEY §8d's per-scheme B/cell (stage-by-stage schedule)
            out["roofline"]["survey_gate"] = survey_gate(SURVEY_BYTES[scheme], cells_local * args.steps, ms4)
        if k8:
            # K8 (stage pairs, the library default for RK4 / explicit midpoint on one GPU): 112 /
            # 32 B/cell, bound by instruction issue and FP64 latency, not HBM -- the roofline is
            # the FP64 pipe (148 SMs x 64 non-FMA ops/clk at the max SM clock) on the
            # algorithmic op count per cell-step (the tile-ring re-evaluations of
            # stage A are not counted); the HBM view stays beside it
            k_ms = out["roofline"]["avg_launch_ms"] * K8_LAUNCHES[scheme]
            ops = K6_OPS[scheme] * cells_local / (k_ms / 1e3) / 1e12 if k_ms else None
            peak_ops = 148 * 64 * 1965e6 / 1e12
            out["kernel"] = "gs_pair_kernel (K8: two chained stages per launch, stage A on the tile + 1 ring)"
            out["roofline"] = {"bound": "alu", "achieved": ops, "peak": peak_ops, "unit": "TFLOP/s (fp64, non-FMA)",
                               "frac": ops / peak_ops if ops else None, "ops_per_cell_step": K6_OPS[scheme],
                               "avg_launch_ms": out["roofline"]["avg_launch_ms"],
                               "hbm": {"achieved": a4, "peak": peak, "unit": "GB/s", "frac": a4 / peak if a4 else None,
                                       "algorithmic_bytes_per_cell_step": out["roofline"]["algorithmic_bytes_per_cell_step"]}}
        h = halo_of(s4, bool(p2p))
        if h:
            out["halo"] = h
        return out

    def k3_leg(scheme):
        # the stage-by-stage kernels (K3, RK_OPT_FUSED_STEP = 0) on the same workload: the
        # HBM-roofline reference the K8 default is measured against
        st.set_option(rk.OPT_FUSED_STEP, 0)
        try:
            out = rk4_leg(args.overlap, scheme, k8_ok=False)
        finally:
            st.set_option(rk.OPT_FUSED_STEP, 3)
        out["kernel"] = "gs_stage_kernel (K3: one stage per launch)"
        return out

    def k6_leg(scheme, mode=1):
        st.set_option(rk.OPT_FUSED_STEP, mode)
        with ClockSampler(local) as clk:
            out = rk4_leg(args.overlap, scheme, k8_ok=False)
        st.set_option(rk.OPT_FUSED_STEP, 3)
        mhz = (getattr(clk, "result", None) or {}).get("sm_mhz") or 1965.0
        peak_ops = 148 * 64 * mhz * 1e6 / 1e12
        ms = out["ms_per_step"]
        k_ms = out["roofline"]["avg_launch_ms"]
        ach = K6_OPS[scheme] * cells_local / (k_ms / 1e3) / 1e12 if k_ms else None
        out["hbm_bytes_per_cell_step"] = out["roofline"]["algorithmic_bytes_per_cell_step"]
        out["roofline"] = {"bound": "alu", "achieved": ach, "peak": peak_ops, "unit": "TFLOP/s (fp64, non-FMA)",
                           "frac": ach / peak_ops if ach else None, "ops_per_cell_step": K6_OPS[scheme],
                           "avg_launch_ms": k_ms}
        out["kernel"] = ("gs_fused_kernel (K6: whole step per launch, temporal blocking over the stages)" if mode == 1 else
                         "gs_ws_kernel (K7: whole step per launch, warp-specialised stage groups, mbarrier hand-off)")
        out["ms_per_step"] = ms
        return out

    def e2e_leg():
        # the same metric through the C-ABI with HOST buffers: every step copies the IC in
        # (pinned H2D, rk_state_set), integrates (rk_integrate_adaptive, incl. its 8-byte
        # error-ratio D2H per try) and copies the result out (pinned D2H, rk_state_get)
        host_in = torch.from_numpy(u0).pin_memory()
        host_out = torch.empty_like(host_in).pin_memory()
        integrate_step(host_in)
        ke = max(1, min(args.steps, 5))
        barrier()
        acc = 0
        ev0.record(stream)
        for _ in range(ke):
            a, _ = integrate_step(host_in)  # H2D of the step's input state + the integration
            acc += a
            st.get(host_out)                # D2H of the step's result
        ev1.record(stream)
        barrier()
        mse = max_over_ranks(ev0.elapsed_time(ev1))
        serial = {"value": cells_total * acc / (mse / 1e3), "unit": "cell-updates/s",
                  "h2d_bytes_per_step": u0.nbytes, "d2h_bytes_per_step": u0.nbytes,
                  "steps": ke, "ms_per_step": mse / ke,
                  "mode": "serial: set (H2D), integrate, get (D2H), one step after the other"}
        try:  # the headline e2e: the same per-step work, two steps in flight
            out = e2e_pipelined(host_in, ke)
        except Exception as exc:  # noqa: BLE001
            return dict(serial, pipelined={"error": f"{type(exc).__name__}: {exc}"})
        out["serial"] = serial
        return out

    def e2e_pipelined(host_in, ke):
        # the same per-step work (H2D of the input, integrate, D2H of the result), two steps in
        # flight: two contexts on their own streams, driven from two host threads (the C-ABI
        # calls release the GIL), so one step's PCIe copies overlap the other's integration
        import threading
        side = [torch.cuda.Stream(local), torch.cuda.Stream(local)]
        ctxs, sts, outs = [], [], []
        for i in range(2):
            c = rk.Context.from_torch_distributed(local, side[i]) if world > 1 else rk.Context(0, 1, local, side[i])
            g = c.grid(n, n, nzg, 2)
            g.set_rhs_gray_scott(h=H)
            g.set_option(rk.OPT_HALO_OVERLAP, args.overlap)
            ctxs.append(c)
            sts.append(g)
            outs.append(torch.empty_like(host_in).pin_memory())
        accs = [0, 0]
        # one integration on the GPU at a time: the other pipeline's D2H + H2D run on the copy
        # engines meanwhile, so the GPU never waits on PCIe and two integrations never split it.
        # The pipelines take strict turns (0, 1, 0, 1, ...), the same order on every rank: with
        # N > 1 each integration runs collectives on its own context's communicator, and a
        # first-come lock could hand rank 0's GPU to pipeline 0 and rank 1's to pipeline 1 --
        # each waiting in a collective for a peer that waits for the lock.
        turn = [0]
        cv = threading.Condition()
        errors = []

        def work(i, k):
            try:
                for _ in range(k):
                    sts[i].set(host_in)
                    with cv:
                        cv.wait_for(lambda: turn[0] % 2 == i or errors)
                    if errors:
                        return
                    try:
                        a, _ = sts[i].integrate_adaptive("dopri5", 0.0, T1, 1.0, TOL, TOL)
                    finally:  # the other pipeline's turn even if this one failed
                        with cv:
                            turn[0] += 1
                            cv.notify_all()
                    sts[i].get(outs[i])
                    accs[i] += a
            except Exception as exc:  # noqa: BLE001 -- re-raised by the caller after the join
                with cv:
                    errors.append(exc)
                    cv.notify_all()

        for i in range(2):
            work(i, 1)
        if errors:
            raise errors[0]
        accs[0] = accs[1] = 0
        kper = max(2, args.steps)  # per pipeline: 2*steps in the timed region (fill / drain amortised)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(side[0])
        side[1].wait_event(e0)
        th = [threading.Thread(target=work, args=(i, kper)) for i in range(2)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errors:
            raise errors[0]
        ej = torch.cuda.Event()
        ej.record(side[1])
        side[0].wait_event(ej)
        e1.record(side[0])
        barrier()
        ms = max_over_ranks(e0.elapsed_time(e1))
        for g in sts:
            g.close()
        for c in ctxs:
            c.close()
        steps = 2 * kper
        return {"value": cells_total * (accs[0] + accs[1]) / (ms / 1e3), "unit": "cell-updates/s",
                "h2d_bytes_per_step": u0.nbytes, "d2h_bytes_per_step": u0.nbytes, "steps": steps,
                "ms_per_step": ms / steps,
                "mode": "two steps in flight (two contexts / streams / host threads, one integration "
                        "on the GPU at a time): one step's H2D + D2H overlap the other's integration"}

    def native_rk4_leg():
        # f4 ablation: RK4 from separate ops, every stage value and k_j
        # through HBM (4 rk_eval_rhs + 4 rk_lincomb launches per step), vs the fused stages
        from paper_2309_05331_b200.ablation import NativeRK4
        st.set(u0_dev)
        nat = NativeRK4(st)
        for _ in range(args.warmup):
            nat.step(1.0)
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            nat.step(1.0)
        ev1.record(stream)
        barrier()
        ms = max_over_ranks(ev0.elapsed_time(ev1))
        nat.close()
        # per cell and step: 4 x (Y or u -> k) + 3 x (u, k -> Y) + (u, k1..k4 -> u), 16 B arrays
        bpc = 4 * 32 + 3 * 48 + 96
        ach = bpc * cells_local * args.steps / (ms / 1e3) / 1e9
        out = {"value": cells_total * args.steps / (ms / 1e3), "ms_per_step": ms / args.steps,
               "scheme": "rk4 unfused (RK_OPT_FUSED_KERNELS = 0: 4 RHS + 4 lincomb launches per step)",
               "algorithmic_bytes_per_cell_step": bpc, "achieved_gbs": ach, "frac_of_peak": ach / peak}
        # the headline integration in the unfused dataflow (Y_i, k_i, u_new, e through HBM)
        st.set_option(rk.OPT_FUSED_KERNELS, 0)
        integrate_step(u0_dev)
        ms_d = []
        for _ in range(max(1, min(args.steps, 3))):
            barrier()
            ev0.record(stream)
            a, r = integrate_step(u0_dev)
            ev1.record(stream)
            barrier()
            ms_d.append(max_over_ranks(ev0.elapsed_time(ev1)))
        st.set_option(rk.OPT_FUSED_KERNELS, 1)
        m = statistics.median(ms_d)
        out["dopri5_adaptive_unfused"] = {"value": cells_total * a / (m / 1e3), "unit": "cell-updates/s",
                                          "ms_per_integration": m, "ms_per_try": m / (a + r), "accepted": a,
                                          "rejected": r}
        return out

    def exp512_leg():
        # f4: the exponential-family workload: 512 x 512 = 262,144
        # independent ODEs du/dt = u, block-split over the ranks (strong scaling), RK4
        n_side = 512
        nv = n_side * n_side
        ve = ctx.vector(nv)
        ve.set_rhs_exponential(1.0)
        ue = rk_inputs.exp_family_u0(n_side)[ve.begin:ve.begin + ve.local].copy()
        out = {"config": {"workload": "exp_family_512^2 (262,144 ODEs, du/dt=u), RK4 dt=1e-3",
                          "partition": f"block x{world}", "scaling": "strong"}}
        for mode, nstep in (("do_step", 200), ("integrate_const", 1000)):
            ve.set(ue)
            if mode == "do_step":
                run = lambda: [ve.do_step("rk4", 0.0, 1e-3) for _ in range(nstep)]  # noqa: E731
            else:
                run = lambda: ve.integrate_const("rk4", 0.0, nstep * 1e-3, 1e-3)  # noqa: E731
            for _ in range(args.warmup):
                run()
            ve.reset_stats()
            barrier()
            ev0.record(stream)
            for _ in range(args.steps):
                run()
            ev1.record(stream)
            barrier()
            ms = max_over_ranks(ev0.elapsed_time(ev1))
            out[mode] = {"value": nv * nstep * args.steps / (ms / 1e3), "unit": "element-updates/s",
                         "ms_per_step": ms / (nstep * args.steps),
                         "gpu_launches_per_step": ve.stats()["kernel_launches"] / (nstep * args.steps)}
        ve.close()
        return out

    def small_configs_leg():
        # f3: the launch-bound configs.  configs[2]: Gray–Scott 64^3 RK4 dt=1,
        # integrate_const 0..20 launched step by step vs replayed from a CUDA graph
        # (RK_OPT_USE_GRAPH); configs[1]: logistic N=1e6 DOPRI5 adaptive tol 1e-8 on [-5, 5]
        # with the host-driven try loop vs the one-launch device loop (RK_OPT_DEVICE_LOOP)
        out = {}
        if world == 1:
            n64 = 64
            g = ctx.grid(n64, n64, n64, 2)
            g.set_rhs_gray_scott(h=H)
            u64 = rk_inputs.gray_scott_ic(n64, n64, n64, seed=42)
            for mode in ("launches", "graph", "persistent"):
                graph = mode == "graph"
                g.set_option(rk.OPT_USE_GRAPH, 1 if graph else 0)
                # persistent: K5, all stages of all steps in one cooperative launch
                g.set_option(rk.OPT_COOP_MAX_CELLS, n64 ** 3 if mode == "persistent" else 0)
                g.set(u64)
                g.integrate_const("rk4", 0.0, 20.0, 1.0)
                ms = []
                for _ in range(max(3, args.steps)):
                    g.set(u64)
                    torch.cuda.synchronize()
                    ev0.record(stream)
                    g.integrate_const("rk4", 0.0, 20.0, 1.0)
                    ev1.record(stream)
                    torch.cuda.synchronize()
                    ms.append(ev0.elapsed_time(ev1))
                m = statistics.median(ms)
                out[{"launches": "gs64_rk4", "graph": "gs64_rk4_graph",
                     "persistent": "gs64_rk4_persistent"}[mode]] = {
                    "value": n64 ** 3 * 20 / (m / 1e3), "unit": "cell-updates/s", "ms_per_step": m / 20,
                    "config": "configs[2]: 64^3, RK4, dt=1, t in [0,20], median of integrate_const calls"}
            # DOPRI5 error control on the same 64^3 grid (tol 1e-6, dt0 = 1, t in [0, 20]): the
            # host-driven try loop over K3 stage launches vs the whole loop in one K5 launch
            g.set_option(rk.OPT_USE_GRAPH, 0)
            for dl in (0, 1):
                g.set_option(rk.OPT_DEVICE_LOOP, dl)
                g.set_option(rk.OPT_COOP_MAX_CELLS, n64 ** 3 if dl else 0)
                ms, tries, acc = [], 0, 0
                for _ in range(max(3, args.steps)):
                    g.set(u64)
                    torch.cuda.synchronize()
                    ev0.record(stream)
                    a, r = g.integrate_adaptive("dopri5", 0.0, 20.0, 1.0, TOL, TOL)
                    ev1.record(stream)
                    torch.cuda.synchronize()
                    ms.append(ev0.elapsed_time(ev1))
                    tries, acc = a + r, a
                m = statistics.median(ms)
                out["gs64_dopri5_adaptive_device_loop" if dl else "gs64_dopri5_adaptive"] = {
                    "value": n64 ** 3 * acc / (m / 1e3), "unit": "cell-updates/s", "ms_per_step": m / acc,
                    "tries": tries, "accepted": acc, "us_per_try": 1e3 * m / tries,
                    "config": "64^3, DOPRI5 tol 1e-6, dt0 1, t in [0,20], median of integrate_adaptive calls"}
            g.close()
            nv = 1000000
            v = ctx.vector(nv)
            v.set_rhs_logistic()
            ul = rk_inputs.logistic_u0(nv)
            for dl in (0, 1):
                v.set_option(rk.OPT_DEVICE_LOOP, dl)
                ms, tries = [], 0
                for _ in range(max(3, args.steps)):
                    v.set(ul)
                    torch.cuda.synchronize()
                    ev0.record(stream)
                    a, r = v.integrate_adaptive("dopri5", -5.0, 5.0, 0.1, 1e-8, 1e-8)
                    ev1.record(stream)
                    torch.cuda.synchronize()
                    ms.append(ev0.elapsed_time(ev1))
                    tries = a + r
                m = statistics.median(ms)
                out["logistic_1e6_dopri5_device_loop" if dl else "logistic_1e6_dopri5"] = {
                    "value": nv * tries / (m / 1e3), "unit": "element-tries/s", "ms_per_step": m / tries,
                    "ms_per_integration": m, "tries": tries,
                    "config": "configs[1]: N=1e6 logistic, DOPRI5 adaptive atol=rtol=1e-8, t in [-5,5], dt0=0.1"}
            v.close()
        return out

    def device_loop_leg():
        # f3: the whole integrate_adaptive as one CUDA-graph launch (RK_OPT_DEVICE_LOOP: no host
        # round trip per try) vs the host-driven try loop, at 512^3 and on the G = 8 strong-
        # scaling share (512 x 512 x 64 slab, one GPU, no exchange), DOPRI5 tol 1e-6, [0, 20]
        out = {}
        for nzl in (n, n // 8):
            g = ctx.grid(n, n, nzl, 2) if nzl != n else st
            if g is not st:
                g.set_rhs_gray_scott(h=H)
            # the G = 8 share holding the middle of the IC cube (non-trivial dynamics)
            ug = u0_dev if g is st else torch.from_numpy(
                rk_inputs.gray_scott_ic(n, n, n, seed=42, z0=(n - nzl) // 2, nzl=nzl, zblocks=1)).cuda(local)
            res = {}
            for dl in (0, 1):
                g.set_option(rk.OPT_DEVICE_LOOP, dl)
                g.set(ug)
                g.integrate_adaptive("dopri5", 0.0, T1, 1.0, TOL, TOL)  # warm-up (and graph build)
                ms, tries, acc = [], 0, 0
                for _ in range(max(3, args.warmup)):
                    g.set(ug)
                    barrier()
                    ev0.record(stream)
                    a, r = g.integrate_adaptive("dopri5", 0.0, T1, 1.0, TOL, TOL)
                    ev1.record(stream)
                    barrier()
                    ms.append(max_over_ranks(ev0.elapsed_time(ev1)))
                    tries, acc = a + r, a
                m = statistics.median(ms)
                res["device_loop" if dl else "host_loop"] = {
                    "value": n * n * nzl * acc / (m / 1e3), "unit": "cell-updates/s", "ms_per_integration": m,
                    "ms_per_try": m / tries, "tries": tries, "accepted": acc}
            g.set_option(rk.OPT_DEVICE_LOOP, 0)
            if g is not st:
                g.close()
            res["speedup"] = res["host_loop"]["ms_per_integration"] / res["device_loop"]["ms_per_integration"]
            out[f"nz{nzl}"] = res
        out["config"] = "DOPRI5 tol 1e-6, t in [0, 20], dt0 1; median of 3 integrate_adaptive calls"
        return out

    def strong_emul_leg():
        # configs[3] on ONE GPU: the per-GPU share of a G-way strong-scaling run (512 x 512 x
        # 512/G slab of the 512^3 IC) through the multi-GPU stage path in loopback mode (pack,
        # ghost planes, interior + overlapped boundary launches; the exchange is NCCL's self
        # send/recv -- or the P2P stores -- on one GPU instead of NVLink).  Compute-side efficiency
        # only: T(512^3) / (G * T(slab)) per try; NVLink time is not in it.  DOPRI5 runs whole
        # integrations over [0, 20] of the slab holding the middle of the IC cube, through three
        # transports / drivers: NCCL + host try loop, P2P + host try loop, P2P + the
        # device-resident graph loop (f3: no host round trip per try); RK4 as do_step.
        out = {}
        variants = (("nccl_host", 0, 0), ("p2p_host", 1, 0), ("p2p_device", 1, 1))
        for G in (1, 2, 4, 8):
            nzl = n // G
            eg = ctx.grid(n, n, nzl, 2)
            eg.set_rhs_gray_scott(h=H)
            eg.set_option(rk.OPT_HALO_LOOPBACK, 1 if G > 1 else 0)
            ue = torch.from_numpy(rk_inputs.gray_scott_ic(n, n, n, seed=42, z0=(n - nzl) // 2, nzl=nzl,
                                                          zblocks=1)).cuda(local)
            res = {}
            for name, p2p, dl in (variants if G > 1 else (("host", 0, 0), ("device", 0, 1))):
                eg.set_option(rk.OPT_HALO_P2P, p2p)
                eg.set_option(rk.OPT_DEVICE_LOOP, dl)
                eg.set(ue)
                eg.integrate_adaptive("dopri5", 0.0, T1, 1.0, TOL, TOL)  # warm-up / graph build
                ms, tries = [], 0
                for _ in range(3):
                    eg.set(ue)
                    barrier()
                    ev0.record(stream)
                    a, r = eg.integrate_adaptive("dopri5", 0.0, T1, 1.0, TOL, TOL)
                    ev1.record(stream)
                    barrier()
                    ms.append(ev0.elapsed_time(ev1))
                    tries = a + r
                m = statistics.median(ms)
                res["dopri5_" + name] = {"ms_per_integration": m, "tries": tries, "ms_per_try": m / tries}
            eg.set_option(rk.OPT_DEVICE_LOOP, 0)
            # RK4: K8 stage pairs on one GPU and over NCCL ghost planes; the P2P transport runs
            # the stage-by-stage kernels (K3), so its efficiency is against K3's G = 1 ("plain_k3")
            for name, p2p in ((("nccl", 0), ("p2p", 1)) if G > 1 else (("plain", 0), ("plain_k3", 0))):
                eg.set_option(rk.OPT_HALO_P2P, p2p)
                eg.set_option(rk.OPT_FUSED_STEP, 0 if name == "plain_k3" else 3)
                eg.set(ue)
                for _ in range(args.warmup):
                    eg.do_step("rk4", 0.0, 1.0)
                barrier()
                ev0.record(stream)
                for _ in range(args.steps):
                    eg.do_step("rk4", 0.0, 1.0)
                ev1.record(stream)
                barrier()
                res["rk4_" + name] = {"ms_per_step": ev0.elapsed_time(ev1) / args.steps}
            eg.set_option(rk.OPT_FUSED_STEP, 3)
            eg.close()
            out[f"G{G}"] = {"nz_per_gpu": nzl, **res}
        t1_dp = out["G1"]["dopri5_host"]["ms_per_try"]
        t1_rk = out["G1"]["rk4_plain"]["ms_per_step"]
        t1_rk3 = out["G1"]["rk4_plain_k3"]["ms_per_step"]
        for G in (2, 4, 8):
            o = out[f"G{G}"]
            for name, _, _ in variants:
                o["dopri5_" + name]["compute_efficiency_per_try"] = t1_dp / (G * o["dopri5_" + name]["ms_per_try"])
            for name, t1 in (("nccl", t1_rk), ("p2p", t1_rk3)):
                o["rk4_" + name]["compute_efficiency"] = t1 / (G * o["rk4_" + name]["ms_per_step"])
        out["config"] = ("per-GPU share of configs[3] (512^3 strong scaling) on one GPU, loopback halo path "
                         "(NCCL self send/recv or P2P stores); DOPRI5 tol 1e-6 integrations over [0, 20]")
        return out

    def strong_leg():
        # configs[3]: 512^3 in total, z-slab over the ranks (strong scaling), DOPRI5 adaptive
        # tol 1e-6 and RK4 dt = 1, as the headline but with nz_local = 512 / N
        sg = ctx.grid(n, n, n, 2)
        sg.set_rhs_gray_scott(h=H)
        sg.set_option(rk.OPT_HALO_OVERLAP, args.overlap)
        us = torch.from_numpy(rk_inputs.gray_scott_ic(n, n, n, seed=42, z0=sg.begin, nzl=sg.local,
                                                      zblocks=1)).cuda(local)
        sg.set(us)
        t, dt = 0.0, 1.0

        def acc_step():
            nonlocal t, dt
            tries = 0
            while True:
                ok, _, dtn = sg.try_step("dopri5", t, dt, TOL, TOL)
                tries += 1
                if ok:
                    t, dt = t + dt, dtn
                    return tries
                dt = dtn
        for _ in range(args.warmup):
            acc_step()
        barrier()
        ev0.record(stream)
        tries = sum(acc_step() for _ in range(args.steps))
        ev1.record(stream)
        barrier()
        ms_a = max_over_ranks(ev0.elapsed_time(ev1))
        sg.set(us)
        for _ in range(args.warmup):
            sg.do_step("rk4", 0.0, 1.0)
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            sg.do_step("rk4", 0.0, 1.0)
        ev1.record(stream)
        barrier()
        ms_r = max_over_ranks(ev0.elapsed_time(ev1))
        sg.close()
        return {"config": {"workload": "gray_scott_512^3_total", "nz_per_gpu": int(sg.local), "scaling": "strong"},
                "dopri5_adaptive": {"value": n ** 3 * args.steps / (ms_a / 1e3), "unit": "cell-updates/s",
                                    "ms_per_step": ms_a / args.steps, "tries": tries},
                "rk4": {"value": n ** 3 * args.steps / (ms_r / 1e3), "unit": "cell-updates/s",
                        "ms_per_step": ms_r / args.steps}}

    def exposed_halo_leg():
        # exposed halo = T(overlap on) - T(no-comm run of the same slab).  N > 1:
        # every rank also runs its own slab as a one-GPU periodic problem (z wraps locally, no
        # exchange) on a private context; N = 1: the loopback halo path against the plain one.
        def rk4_ms(state):
            state.set_option(rk.OPT_HALO_OVERLAP, 1)
            for _ in range(args.warmup):
                state.do_step("rk4", 0.0, 1.0)
            barrier()
            ev0.record(stream)
            for k in range(args.steps):
                state.do_step("rk4", float(k), 1.0)
            ev1.record(stream)
            barrier()
            return max_over_ranks(ev0.elapsed_time(ev1)) / args.steps
        st.set(u0_dev)
        if world == 1:
            st.set_option(rk.OPT_HALO_LOOPBACK, 1)
        t_on = rk4_ms(st)
        st.set_option(rk.OPT_HALO_LOOPBACK, 0)
        c1 = rk.Context(0, 1, local, stream)
        solo = c1.grid(n, n, int(st.local), 2)
        solo.set_rhs_gray_scott(h=H)
        solo.set(u0_dev)
        t_off = rk4_ms(solo)
        solo.close()
        c1.close()
        return {"scheme": "rk4 (K8 stage pairs on both sides: on the slab path with 2-deep ghost planes "
                          "exchanged before each pair, not overlapped)",
                "ms_per_step_halo_overlapped": t_on, "ms_per_step_no_comm": t_off,
                "exposed_halo_ms_per_step": t_on - t_off, "exposed_frac": (t_on - t_off) / t_off,
                "halo_path": "nccl send/recv" if world > 1 else "loopback (one GPU)"}

    def run_leg(fn, *a):
        # an extra leg that fails reports its error instead of losing the headline line
        try:
            return fn(*a)
        except Exception as exc:  # noqa: BLE001
            return {"error": f"{type(exc).__name__}: {exc}"}

    line = adaptive_leg() if "adaptive" in legs else {}
    extra = {}
    if "rk4" in legs:
        extra["rk4"] = run_leg(rk4_leg, args.overlap)
        r4 = extra["rk4"]
        if line and "roofline" in r4:
            # north_star's second target workload, kept inside `roofline` (the driver's parsed
            # record keeps this object but not `extra`)
            rf = r4["roofline"]
            line["roofline"]["rk4_512"] = {
                "workload": "gray_scott_rk4_dt1_512^3_per_gpu (do_step x K)", "value": r4["value"],
                "unit": "cell-updates/s", "ms_per_step": r4["ms_per_step"], "kernel": r4.get("kernel", "K3"),
                "bound": rf["bound"], "achieved": rf["achieved"], "peak": rf.get("peak"), "unit_roofline": rf.get("unit"),
                "frac": rf["frac"]}
            if "hbm" in rf:
                line["roofline"]["rk4_512"]["hbm"] = rf["hbm"]
            else:
                line["roofline"]["rk4_512"]["algorithmic_bytes_per_cell_step"] = rf["algorithmic_bytes_per_cell_step"]
                line["roofline"]["rk4_512"]["traffic"] = rf["traffic"]
    if "rk4_k3" in legs and world == 1:
        extra["rk4_k3"] = run_leg(k3_leg, "rk4")
        if line and "rk4_512" in line.get("roofline", {}) and "ms_per_step" in extra["rk4_k3"]:
            k3 = extra["rk4_k3"]
            line["roofline"]["rk4_512"]["stage_by_stage"] = {
                "kernel": "K3", "ms_per_step": k3["ms_per_step"], "frac_hbm": k3["roofline"]["frac"],
                "algorithmic_bytes_per_cell_step": k3["roofline"]["algorithmic_bytes_per_cell_step"]}
    if "try_loop" in legs:
        extra["dopri5_try_loop"] = run_leg(try_loop_leg)
    if "repeats" in legs:
        # each config 3 times, mean and min (the headline line is the first run)
        def rep(fn, *a):
            try:
                return [fn(*a)["ms_per_step"] for _ in range(2)]
            except Exception:  # noqa: BLE001
                return []
        rp = {}
        if "adaptive" in legs and line:
            ms = [line["ms_per_step"]] + rep(adaptive_leg)
            rp["dopri5_adaptive_ms_per_step"] = {"runs": ms, "mean": sum(ms) / len(ms), "min": min(ms)}
        if "rk4" in legs and "ms_per_step" in extra.get("rk4", {}):
            ms = [extra["rk4"]["ms_per_step"]] + rep(rk4_leg, args.overlap)
            rp["rk4_ms_per_step"] = {"runs": ms, "mean": sum(ms) / len(ms), "min": min(ms)}
        extra["repeats"] = rp
    if "rk4" in legs:
        if world > 1:
            extra["rk4_overlap_off"] = run_leg(rk4_leg, 0)
    if "halo" in legs:
        # f3: the halo machinery on RK4 -- N = 1: loopback self-exchange through NCCL's path
        # (device copy) and through the P2P path; N > 1: P2P stores over NVLink vs NCCL above
        if world == 1:
            extra["rk4_loopback_nccl"] = run_leg(rk4_leg, args.overlap, "rk4", 0, 1)
            extra["rk4_loopback_p2p"] = run_leg(rk4_leg, args.overlap, "rk4", 1, 1)
        elif "p2p" in legs:  # opt-in at N > 1: needs CUDA IPC between the rank processes
            extra["rk4_p2p"] = run_leg(rk4_leg, args.overlap, "rk4", 1, 0)
    if "exposed" in legs:
        extra["exposed_halo"] = run_leg(exposed_halo_leg)
    if "device_loop" in legs and world == 1:
        extra["device_loop"] = run_leg(device_loop_leg)
    if "strong_emul" in legs and world == 1:
        extra["strong_emul"] = run_leg(strong_emul_leg)
    if "strong" in legs and world > 1:
        extra["strong"] = run_leg(strong_leg)
    if "rk4_native" in legs:
        extra["rk4_native"] = run_leg(native_rk4_leg)
    if "midpoint_k3" in legs and world == 1:
        extra["midpoint_k3"] = run_leg(k3_leg, "midpoint")
    for sch in ("rk4", "midpoint", "modified_midpoint"):  # --legs rk4_k6,rk4_k7,...
        for mode in (1, 2):
            leg = f"{sch}_k{5 + mode}"
            if leg in legs and world == 1:
                extra[leg] = run_leg(k6_leg, sch, mode)
    if "exp512" in legs:
        extra["exp512"] = run_leg(exp512_leg)
    if "small" in legs:
        extra["small_configs"] = run_leg(small_configs_leg)
    for sch in (("euler", "midpoint", "modified_midpoint", "cash_karp54", "dopri5", "rkf78")
                + tuple(f"ab{k}" for k in range(1, 9))
                + tuple(f"abm{k}" for k in range(1, 9))):
        # scheme sweep (configs[4])
        if sch in legs:
            extra[sch] = run_leg(rk4_leg, args.overlap, sch)
    if extra:
        line["extra"] = extra
    if "e2e" in legs:
        line["e2e"] = e2e_leg()
    if "cpu" in legs and rank == 0 and world == 1:
        line["cpu_baseline"] = cpu_baseline()
    if "cpu_full" in legs and rank == 0 and world == 1:  # opt-in: ~1 min, ~25 GB host RAM
        line.setdefault("cpu_baseline", {})["full_512"] = oracle_full_512()
    if rank == 0:
        print(json.dumps(line), flush=True)
    st.close()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
