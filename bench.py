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
    """nvidia-smi clock / throttle sampling during the timed region (B200_PROFILING.md recipe)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
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

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [s.strip() for s in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(config: str, seconds_hint: float = 30.0) -> dict:
    """The float64 oracle (as it stands) on the host cores: fwd+grad of ONE signal of `config`."""
    import torch
    from oracle.jtfs import Oracle
    cores = torch.get_num_threads()
    o = Oracle(plan_args(CONFIGS[config]))
    x = batch(config, 1)
    y = batch(config, 1, which="y")
    St = o.forward(x)                    # target coefficients: not part of the timed step
    t0 = time.perf_counter()
    o.loss_grad(y, St)
    dt = time.perf_counter() - t0
    N = CONFIGS[config]["N"]
    return {"value": N / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"1 signal of {config} (N={N}), float64 forward+loss+gradient, {dt:.1f} s"}


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
    St = o.forward(x)
    # one reference step = fwd+grad of ONE signal (~1 min on 16 cores); capped at 2 steps so the
    # arm ends within a few minutes whatever --steps says (reported as "steps"); no warm-up steps: the
    # float64 numpy oracle has no JIT or device state to warm (reported as "warmup": 0)
    steps = max(1, min(args.steps, 2))
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        o.loss_grad(y, St)
        times.append(time.perf_counter() - t0)
    dt = float(np.sum(times))
    value = steps * cfg["N"] / dt
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": steps, "warmup": 0, "ms_per_step": 1000 * dt / steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {_describe(args.config)}; reference step = 1 signal"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": torch.get_num_threads(), "kind": "oracle",
                             "sample": f"1 signal of {args.config} per step (float64 oracle, host cores)"},
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
    y0 = torch.from_numpy(batch(args.config, B, which="y")).to(dev)
    St = plan.forward(x)
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
    return {"steps": args.metamer, "steps_per_s": args.metamer / (ms / 1000.0), "ms_per_step": ms / args.metamer,
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
    ap.add_argument("--config", default="c2")
    ap.add_argument("--batch", type=int, default=None, help="signals per rank (default: config batch)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--metamer", type=int, default=0,
                    help="also run this many metamer_step iterations (BASELINE configs[2]: c3, 100) from white-noise "
                         "init and report steps/s and the loss curve under the 'metamer' key")
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
    # per-group batch: independent signals (weak scaling); target S(x) computed once, untimed
    x = torch.from_numpy(batch(args.config, B, start=group_id * B)).to(dev)
    y = torch.from_numpy(batch(args.config, B, which="y", start=group_id * B)).to(dev)
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
            dj.loss_grad(y, St)
        else:
            plan.loss_grad(y, St, loss=loss, grad=grad, ws=ws)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(lrank)
    clocks.start()
    plan.prof_enable(True)
    n0 = plan.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    launches = plan.launch_count() - n0
    plan.prof_enable(False)
    prof = {"joint_fwd": plan.prof_read(0), "joint_bwd": plan.prof_read(2)}
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = n_groups * B * cfg["N"] * args.steps / (ms / 1000.0)

    # end-to-end through the host-buffer C-ABI call (pinned host memory, copies inside)
    e2e = None
    if not args.no_e2e and ps == 1:
        yh = torch.from_numpy(batch(args.config, B, which="y", start=rank * B)).pin_memory()
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
        e2e = {"value": n_groups * B * cfg["N"] * args.steps / (hms / 1000.0), "unit": UNIT,
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
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.config}: {_describe(args.config)} per rank",
                   "l2": "per-step working set > 126 MB L2 (no flush needed)",
                   "micro_batch": int(mb), "parallelism": f"batch{n_groups}xpath{ps}"},
        "roofline": roof,
        "clocks": clk, "gpu_launches": int(launches), "gpu_launches_per_step": launches / args.steps,
    }
    if e2e:
        line["e2e"] = e2e
    if args.metamer > 0:
        line["metamer"] = run_metamer(plan, args, dev)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
