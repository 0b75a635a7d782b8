#!/usr/bin/env python
"""bench.py — JTFS forward+gradient throughput on B200 (BASELINE.json metric).

python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A step = one jtfs_loss_grad over the rank's batch (forward Eqs.2-4, Euclidean loss, dE/dy; the
whole §8(a) hot path A1-A9). Weak scaling: every rank processes its own batch of the config
(independent signals, no data-path collective). Inputs are resident in HBM when the timed
region starts; the per-step working set (>1 GB at c2) exceeds the 126 MB L2, so no extra flush.
value = samples processed by all ranks / (max over ranks of the device time of K steps).
e2e = the same metric through jtfs_loss_grad_host (pinned host buffers, H2D + D2H inside the
timed region). `--impl reference` times the float64 CPU oracle (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import CONFIGS, plan_args, batch  # noqa: E402

METRIC = "JTFS fwd+grad audio samples/s"
UNIT = "samples/s"
FP32_LANES_PER_SM = 128
N_SM = 148


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0, "fallback": True}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    lrank = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, lrank


class Clocks:
    """nvidia-smi clock / throttle sampling (B200_PROFILING.md recipe). The sampler starts before the
    warm-up steps (nvidia-smi needs ~0.1-0.3 s to emit its first line) and every line carries a timestamp;
    stop(t0, t1) keeps the samples inside the timed region [t0, t1] (host wall clock), or, for a timed
    region shorter than the 200 ms sampling period, the samples nearest to it (flagged)."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = f"/tmp/jtfs_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self, t0: float | None = None, t1: float | None = None) -> dict:
        import datetime
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = []
        for line in open(self.path):
            f = [s.strip() for s in line.split(",")]
            if len(f) < 10:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(f[2]), float(f[3]), [n for n, v in zip(names, f[6:10]) if v.lower() == "active"]))
            except ValueError:
                continue
        inside = [r for r in rows if t0 is None or (t0 - 0.05 <= r[0] <= t1 + 0.05)]
        nearest = False
        if not inside and rows and t0 is not None:
            mid = 0.5 * (t0 + t1)
            inside = sorted(rows, key=lambda r: abs(r[0] - mid))[:2]
            nearest = True
        sm = [r[1] for r in inside]
        reasons = sorted({n for r in inside for n in r[3]})
        out = {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": inside[-1][2] if inside else None,
               "reasons": reasons, "samples": len(inside)}
        if nearest:
            out["note"] = "timed region shorter than the 200 ms sampling period: nearest samples"
        return out


def _oracle_sample(config: str, o, x, y):
    """Time the float64 oracle (as it stands) on a BOUNDED sample of one signal's fwd+grad and return
    (seconds for the whole signal, description). c1/c2: the whole signal is timed. c3-c5 (minutes per
    signal on the host): two timed pieces -- layer 1 + order 1 (loss restricted to order 1) and the same
    plus the one second-order block whose column count is nearest 2^14 -- and the whole signal is
    extrapolated as t0 + (t1 - t0) * sum_b T2_b / T2_sample (the oracle's per-block cost is its joint
    stage, proportional to the block's time columns: one P-point FFT per column and filter)."""
    p = o.plan
    if config in ("c1", "c2"):
        St = o.forward(x)
        t0 = time.perf_counter()
        o.loss_grad(y, St)
        dt = time.perf_counter() - t0
        return dt, f"1 signal of {config} (N={p.N}), float64 forward+loss+gradient, {dt:.1f} s measured"
    T2 = [p.N_pad >> b.s2 for b in p.blocks]
    bs = min(range(len(T2)), key=lambda i: abs(np.log2(T2[i]) - 14))
    St = o.forward(x, blocks=[bs])
    t = time.perf_counter()
    o.loss_grad_subset(y, St, [])
    t0 = time.perf_counter() - t
    t = time.perf_counter()
    o.loss_grad_subset(y, St, [bs])
    t1 = time.perf_counter() - t
    dt = t0 + max(t1 - t0, 0.0) * sum(T2) / T2[bs]
    return dt, (f"1 signal of {config} (N={p.N}): layer 1 + order 1 measured {t0:.1f} s, + block {bs} "
                f"({T2[bs]} of {sum(T2)} second-order columns) {t1:.1f} s; whole signal EXTRAPOLATED "
                f"by column count to {dt:.0f} s")


def cpu_baseline(config: str) -> dict:
    """The float64 oracle (as it stands) on the host cores, one signal of `config` (bounded sample)."""
    import torch
    from oracle.jtfs import Oracle
    o = Oracle(plan_args(CONFIGS[config]))
    x = batch(config, 1)
    y = batch(config, 1, which="y")
    dt, what = _oracle_sample(config, o, x, y)
    N = CONFIGS[config]["N"]
    return {"value": N / dt, "unit": UNIT, "cores": torch.get_num_threads(), "kind": "oracle", "sample": what}


def run_reference(args) -> None:
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import torch
    from oracle.jtfs import Oracle
    cfg = CONFIGS[args.config]
    o = Oracle(plan_args(cfg))
    x = batch(args.config, 1)
    y = batch(args.config, 1, which="y")
    # one reference step = the bounded sample of one signal's fwd+grad (_oracle_sample); capped at 2
    # steps so the arm ends within a few minutes whatever --steps says (reported as "steps"); no warm-up
    # steps: the float64 oracle has no JIT or device state to warm (reported as "warmup": 0)
    steps = max(1, min(args.steps, 2))
    times, what = [], ""
    for _ in range(steps):
        dt, what = _oracle_sample(args.config, o, x, y)
        times.append(dt)
    dt = float(np.sum(times))
    value = steps * cfg["N"] / dt
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": steps, "warmup": 0, "ms_per_step": 1000 * dt / steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {_describe(args.config)}; reference step = 1 signal"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": torch.get_num_threads(), "kind": "oracle",
                             "sample": what},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_metamer(plan, args, dev) -> dict:
    """Metamer synthesis: y0 = white noise at the target's RMS, then
    --metamer bold-driver momentum steps (m = 0.9, mu0 = 0.1), all on the device. Reports steps/s (CUDA
    events around the loop) and the mean loss every 10 steps."""
    import torch
    cfg = CONFIGS[args.config]
    B = args.batch or cfg["B"]
    x = torch.from_numpy(batch(args.config, B)).to(dev)
    St = plan.forward(x)
    if args.metamer_init == "colored":   # PAPER.md:123 (reading R25), jtfs_colored_noise
        y0 = plan.colored_noise(St, seed=500000 + 1000 * int(args.config[1:]))
    else:                                # BASELINE configs[2]: Gaussian-noise init at the target's RMS
        y0 = torch.from_numpy(batch(args.config, B, which="y")).to(dev)
    st = plan.metamer_state(y0)
    ws = plan.workspace(B, True, dev)
    curve = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for it in range(args.metamer):
        plan.metamer_step(st, St, ws=ws)
        if it % 10 == 0 or it == args.metamer - 1:
            curve.append([it, float(st["loss"].mean())])   # host read: outside the timed work's critical path
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return {"init": args.metamer_init, "steps": args.metamer, "steps_per_s": args.metamer / (ms / 1000.0),
            "ms_per_step": ms / args.metamer,
            "batch": B, "loss_curve_mean": curve, "final_over_initial": curve[-1][1] / max(curve[0][1], 1e-30),
            "accepted_last": int(st["accepted"].sum())}


def _describe(c: str) -> str:
    d = CONFIGS[c]
    return (f"B={d['B']} N={d['N']} J={d['J']} Q={d['Q']} J_fr={d['J_fr']} Q_fr={d['Q_fr']} "
            f"T={d['T']} F={d['F']}")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", help="BASELINE config (default c4 = configs[3], 'Throughput', "
                                                   "the largest single-GPU config)")
    ap.add_argument("--batch", type=int, default=None, help="signals per rank (default: config batch)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", action="store_true", help="also time the step replayed from a CUDA graph")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: split the config's batch over the batch groups (c5: B = 256 over G)")
    ap.add_argument("--no-forward", action="store_true", help="skip the forward-only (analysis) measurement")
    ap.add_argument("--metamer", type=int, default=0,
                    help="also run this many metamer_step iterations (BASELINE configs[2]: c3, 100) from white-noise "
                         "init and report steps/s and the loss curve under the 'metamer' key")
    ap.add_argument("--metamer-init", default="white", choices=["white", "colored"],
                    help="metamer y0: white Gaussian noise at the target's RMS (BASELINE c3) or the paper's colored "
                         "noise matched to S1 x (jtfs_colored_noise)")
    ap.add_argument("--path-shards", type=int, default=1,
                    help="ranks per path group (order-2 units split, dE/dx all-reduced over NVLink)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist
    from paper_2602_11896_b200 import Plan

    world, rank, lrank = dist_env()
    torch.cuda.set_device(lrank)
    dev = torch.device("cuda", lrank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[args.config]
    B = args.batch or cfg["B"]
    plan = Plan(*plan_args(cfg))
    stream = torch.cuda.current_stream()
    plan.prepare(stream)
    ps = max(1, args.path_shards)
    group_id = rank // ps                     # batch group (signals) of this rank
    n_groups = world // ps
    if args.strong:
        # strong scaling (BASELINE c5: "batch 256 ... at 1/2/4/8 GPUs"): the config's batch is split
        # over the batch groups (contiguous, balanced), the total work is fixed
        from paper_2602_11896_b200.dist import batch_slice
        sl = batch_slice(B, n_groups, group_id)
        start, B_total, B = sl.start, B, sl.stop - sl.start
    else:
        # weak scaling: every batch group processes its own batch of the config (independent signals)
        start, B_total = group_id * B, n_groups * B
    # target S(x) computed once, untimed
    x = torch.from_numpy(batch(args.config, B, start=start)).to(dev)
    y = torch.from_numpy(batch(args.config, B, which="y", start=start)).to(dev)
    St = plan.forward(x)
    ws = plan.workspace(B, True, dev)
    loss = torch.empty(B, device=dev)
    grad = torch.empty_like(y)
    mb = ws.numel() // plan.workspace_size(1, True)
    if ps > 1:
        from paper_2602_11896_b200.dist import DistJTFS
        dj = DistJTFS(plan, path_shards=ps,
                      compute=lambda yy, SS, s, n: plan.loss_grad(yy, SS, shard=s, n_shards=n, loss=loss,
                                                                  grad=grad, ws=ws))

    def step():
        if ps > 1:
            dj.loss_grad(y, St, chunk=mb)   # all_reduce of micro-batch i overlaps micro-batch i+1
        else:
            plan.loss_grad(y, St, loss=loss, grad=grad, ws=ws)

    clocks = Clocks(lrank)
    clocks.start()
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    plan.prof_enable(True)
    n0 = plan.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_wall0 = time.time()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    t_wall1 = time.time()
    ms = e0.elapsed_time(e1)
    launches = plan.launch_count() - n0
    plan.prof_enable(False)
    prof = {"joint_fwd": plan.prof_read(0), "joint_bwd": plan.prof_read(2)}
    clk = clocks.stop(t_wall0, t_wall1)
    if world > 1:
        dist.barrier()
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = B_total * cfg["N"] * args.steps / (ms / 1000.0)

    # CUDA-graph replay of the same step (launch-latency-bound configs, c1: SURVEY §8(d)); the library
    # only enqueues (no host sync inside jtfs_loss_grad), so one step captures whole, side streams included
    graph = None
    if args.graph and ps == 1:
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(stream)
        with torch.cuda.stream(cs):
            plan.loss_grad(y, St, loss=loss, grad=grad, ws=ws)      # warm the capture stream
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            plan.loss_grad(y, St, loss=loss, grad=grad, ws=ws)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            g.replay()
        g1.record(stream)
        torch.cuda.synchronize()
        gms = g0.elapsed_time(g1)
        graph = {"ms_per_step": gms / args.steps, "ms_per_step_eager": ms / args.steps,
                 "value": B_total * cfg["N"] * args.steps / (gms / 1000.0), "unit": UNIT,
                 "what": "one jtfs_loss_grad captured in a CUDA graph (all its launches), replayed"}

    # forward-only analysis throughput (NEXT-2): jtfs_forward over the same batch
    fo_ms = None
    if not args.no_forward:
        Sf = torch.empty_like(St)
        for _ in range(2):
            plan.forward(y, out=Sf, ws=ws)
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        f0.record(stream)
        for _ in range(args.steps):
            plan.forward(y, out=Sf, ws=ws)
        f1.record(stream)
        torch.cuda.synchronize()
        fo_ms = f0.elapsed_time(f1)
        if world > 1:
            t = torch.tensor([fo_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            fo_ms = float(t.item())

    # end-to-end through the host-buffer C-ABI call (pinned host memory, copies inside)
    e2e = None
    if not args.no_e2e and ps == 1:
        yh = torch.from_numpy(batch(args.config, B, which="y", start=start)).pin_memory()
        Sth = St.cpu().pin_memory()
        wsh = plan.workspace_host(B, dev)
        for _ in range(2):
            plan.loss_grad_host(yh.numpy(), Sth.numpy(), ws=wsh)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        h0 = torch.cuda.Event(enable_timing=True)
        h1 = torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        for _ in range(args.steps):
            plan.loss_grad_host(yh.numpy(), Sth.numpy(), ws=wsh)
        h1.record(stream)
        torch.cuda.synchronize()
        hms = h0.elapsed_time(h1)
        if world > 1:
            t = torch.tensor([hms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            hms = float(t.item())
        del wsh
        e2e = {"value": B_total * cfg["N"] * args.steps / (hms / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": int(B * cfg["N"] * 4 + B * plan.n_coef * 4),
               "d2h_bytes_per_step": int(B * 4 + B * cfg["N"] * 4)}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    pk = peaks()
    cost = plan.cost()
    clock_mhz = float(pk.get("sm_max_mhz", 1965.0))
    # peaks: FP32 lanes from the guide's unit counts at the max SM clock; TF32 dense
    # = measured bf16 burst x nominal tf32/bf16 ratio (1.1/2.25); hi/lo 3xTF32 executes 3 MMAs
    fp32_peak = N_SM * FP32_LANES_PER_SM * 2 * clock_mhz * 1e6 / 1e12
    tf32_peak = float(pk.get("bf16_tflops", 1590.0)) * (1.1 / 2.25)
    # Joint-stage groups: each group = the tensor-core launches (3xTF32 contraction) and
    # the FFT-route launch (FP32 CUDA cores) running concurrently. Roofline = the group's ideal time
    # (tensor flops x3 / TF32 peak + FFT-route flops / FP32 peak) over its measured time; "achieved" is
    # the same fraction expressed in TF32-equivalent TFLOP/s against the TF32 peak.
    kern = {}
    for k, (kms, kn) in prof.items():
        if kn == 0:
            continue
        d = "fwd" if k == "joint_fwd" else "bwd"
        tc_fl = cost[d + "_tc_flops"] * B
        ff_fl = cost[d + "_fft_flops"] * B
        t = kms / 1000.0                                   # seconds, all launches of the timed steps
        ideal = args.steps * (3.0 * tc_fl / (tf32_peak * 1e12) + ff_fl / (fp32_peak * 1e12))
        frac = ideal / t
        kern[k] = {"ms_per_step": kms / args.steps, "bound": "tensor", "achieved": frac * tf32_peak,
                   "peak": tf32_peak, "unit": "TFLOP/s", "frac": frac,
                   "tc_tflops_per_step": 3.0 * tc_fl / 1e12, "fft_tflops_per_step": ff_fl / 1e12,
                   "ideal_ms_per_step": 1000.0 * ideal / args.steps}
    dom = max(kern, key=lambda k: kern[k]["ms_per_step"]) if kern else None
    roof = dict(kern[dom]) if dom else {}
    # DRAM traffic of the dominant group per step, from the committed ncu --set full capture of the same
    # command (tools/gpu_session.sh traffic -> profiles/traffic_<config>.json), when one exists
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if dom and os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            traffic = {"bytes_per_step": tj[dom]["dram_bytes_per_step"],
                       "bytes_per_step_per_signal": tj[dom]["dram_bytes_per_step"] / B,
                       "source": os.path.relpath(tpath, ROOT)}
        except Exception:
            traffic = None
    roof.update({"kernel": {"joint_bwd": "k_joint_bwd_tc + k_joint_bwd_fft (concurrent)",
                            "joint_fwd": "k_joint_fwd_tc + k_joint_fwd_fft (concurrent)"}.get(dom, dom),
                 "traffic": traffic, "share_of_step": roof.get("ms_per_step", 0) / (ms / args.steps) if ms else None,
                 "peak_note": ("TF32 dense = measured bf16 %.0f TF x 1.1/2.25 (guide nominal ratio); 3xTF32 "
                               "counts 3 MMAs; FFT route against FP32 = 148 SM x 128 lanes x 2 x %.0f MHz, "
                               "folded into TF32-equivalent time" % (float(pk.get("bf16_tflops", 1590.0)), clock_mhz)),
                 "joint_kernels": kern})
    # clock-true TF32 rate: a kind::tf32 M128 N128 K8 MMA takes N/2 = 64 cycles per SM (DESIGN.md §6,
    # tools/ubench/tmem_mma.cu) -> 4096 flop/cycle/SM at the SM clock measured during the timed region
    f_run = clk.get("sm_mhz") or clock_mhz
    tf32_clock_true = 4096.0 * N_SM * f_run * 1e6 / 1e12
    if dom:
        roof["tf32_clock_true_tflops"] = tf32_clock_true
        roof["frac_vs_tf32_clock_true"] = roof["achieved"] / tf32_clock_true
    # Whole-path roofline: sum over the stages of max(bytes/BW, flops/peak) over the step.
    # Joint stages: their ideal (tensor-bound) time; everything else: algorithmic HBM bytes (SURVEY App. B,
    # fused design: x, X_hat r/w, U1_hat w + 2 r, Y2 w + r fwd, Y2 r + g_Y2 w/r bwd, g_hat_U1, g_hat_x, g)
    # at the measured copy bandwidth.
    hbm_peak = float(pk.get("hbm_gbs", 6545.3))
    sL1, sY2 = plan._sumL1(), plan._sumY2()
    Np = plan.info.N_pad
    alg_bytes_sig = 8 * cfg["N"] + 16 * Np + 40 * sL1 + 40 * sY2
    joint_bytes_sig = cost["joint_hbm_bytes"]
    other_bytes = B * max(alg_bytes_sig - joint_bytes_sig, 0.0)
    step_ms = ms / args.steps
    ideal_joint_ms = sum(kern[k]["ideal_ms_per_step"] for k in kern)
    ideal_other_ms = 1000.0 * other_bytes / (hbm_peak * 1e9)
    path = {"ideal_ms_per_step": ideal_joint_ms + ideal_other_ms, "ms_per_step": step_ms,
            "frac": (ideal_joint_ms + ideal_other_ms) / step_ms, "ideal_joint_ms": ideal_joint_ms,
            "ideal_hbm_ms": ideal_other_ms,
            "joint_ms_measured": sum(kern[k]["ms_per_step"] for k in kern),
            "rest_ms_measured": step_ms - sum(kern[k]["ms_per_step"] for k in kern)}
    # achieved HBM GB/s vs peak (BASELINE metric): algorithmic bytes of the whole path per step over the
    # step time, and the DRAM bytes ncu measured for one step of the same command when committed
    # (profiles/dram_step_<config>.json, tools/ncu_dram.py)
    hbm = {"algorithmic_bytes_per_step": B * alg_bytes_sig, "achieved_gbs": B * alg_bytes_sig / (step_ms * 1e6),
           "peak_gbs": hbm_peak, "frac": B * alg_bytes_sig / (step_ms * 1e6) / hbm_peak,
           "bytes_per_sample": alg_bytes_sig / cfg["N"]}
    dpath = os.path.join(ROOT, "profiles", f"dram_step_{args.config}.json")
    if os.path.exists(dpath):
        try:
            dj = json.load(open(dpath))
            hbm["dram_bytes_per_step_ncu"] = dj["dram_bytes_per_step"] * B / dj.get("batch", B)
            hbm["dram_gbs_ncu_over_step"] = hbm["dram_bytes_per_step_ncu"] / (step_ms * 1e6)
            hbm["dram_source"] = os.path.relpath(dpath, ROOT)
        except Exception:
            pass
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.config}: {_describe(args.config)}" + (" split over ranks" if args.strong
                                                                             else " per batch group"),
                   "l2": "per-step working set > 126 MB L2 (no flush needed)",
                   "micro_batch": int(mb), "parallelism": f"batch{n_groups}xpath{ps}"},
        "roofline": roof, "path_roofline": path, "hbm": hbm,
        "clocks": clk, "gpu_launches": int(launches), "gpu_launches_per_step": launches / args.steps,
    }
    if e2e:
        line["e2e"] = e2e
    if graph:
        line["cuda_graph"] = graph
    if fo_ms is not None:
        line["forward_only"] = {"value": B_total * cfg["N"] * args.steps / (fo_ms / 1000.0), "unit": UNIT,
                                "ms_per_step": fo_ms / args.steps,
                                "what": "jtfs_forward over the same batch (analysis workload, NEXT-2)"}
    if args.metamer > 0:
        line["metamer"] = run_metamer(plan, args, dev)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
