#!/usr/bin/env python
"""LF-MMI loss+grad throughput (frames/s) on B200 — the BASELINE.json metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config wsj_mono]
    python bench.py --impl reference ...     # reference CPU implementation arm

One step = one LF-MMI loss + gradient over one synthetic batch of the named
config (numerator pass + denominator pass, forward + backward + posteriors +
grad), inputs resident in HBM, graphs uploaded once.  Between timed steps L2
is flushed (a 512 MiB write, outside the timed events).  Multi-GPU: one
process per GPU (torchrun), each rank runs its own batch (seed = rank) —
weak scaling — and the three scalar totals are all-reduced over NCCL inside
the step; time is the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary.json")
METRIC = "frames/sec LF-MMI loss+grad (den+num fwd-bwd) at 1/2/4/8 B200; % HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="wsj_mono")
    ap.add_argument("--batch", type=int, default=None, help="override B of the config")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no clocks/cpu)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ helpers
def algorithmic_bytes(lengths, D, S_den, I_den, num_S, num_I):
    """compulsory fp32 HBM bytes of one loss+grad step."""
    frames = int(np.sum(lengths))
    return (frames * (4 * D + 4 * D + 8 * S_den) + 24 * I_den + 12 * S_den
            + int(np.sum(24 * np.asarray(num_I) + 12 * np.asarray(num_S))))


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(
                        ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                         "--format=csv,noheader,nounits"], capture_output=True, text=True,
                        timeout=5).stdout.strip()
                    if out:
                        self.rows.append([c.strip() for c in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


# ---------------------------------------------------------- CPU baselines
def reference_module():
    """The unmodified reference (chainloss 0.1.0) installed in baseline/_ref, if present."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "chainloss")):
        return None
    os.environ.setdefault("NUMBA_NUM_THREADS", str(os.cpu_count() or 1))
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_lfmmi")
    os.environ.setdefault("PYTHONPYCACHEPREFIX", "/tmp/pyc_lfmmi")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import chainloss

    return chainloss


def cpu_reference_run(w, steps, warmup, sample_b=None):
    """Time the reference's own chain_loss (or the oracle port) on host cores.

    Returns (frames_per_s, info dict).  Graph construction and make_batch are
    excluded; best-of-steps after warm-up.
    """
    C = reference_module()
    if sample_b is not None:
        idx = list(range(min(sample_b, len(w.seqs))))
        w = type(w)(w.name, w.seed, w.S, w.I, w.D, w.lengths[idx], [w.seqs[i] for i in idx],
                    w.den, [w.num_phones[i] for i in idx])
    frames = w.total_frames
    if C is not None:
        import numba

        batch, nums, den = w.build(C)
        opts = C.FBOptions()
        times = []
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            C.chain_loss(batch, nums, den, opts)
            dt = time.perf_counter() - t0
            if i >= warmup:
                times.append(dt)
        best = min(times)
        return frames / best, {"kind": "reference", "cores": int(numba.get_num_threads()),
                               "times_s": times, "frames": frames, "B": len(w.seqs)}
    from oracle import oracle as O
    import paper_2005_09824_b200 as P

    batch, nums, den = w.build(P)
    times = []
    for i in range(max(1, warmup) + steps):
        t0 = time.perf_counter()
        O.chain_loss(batch, nums, den)
        dt = time.perf_counter() - t0
        if i >= max(1, warmup):
            times.append(dt)
    return frames / min(times), {"kind": "port", "cores": 1, "times_s": times, "frames": frames,
                                 "B": len(w.seqs)}


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2005_09824_b200 import synth

    w = synth.make_workload(args.config, seed=0, batch_size=args.batch)
    steps = max(1, args.steps)
    # Bound the run: sample the batch so one step is ~<1.5 s of CPU work.
    sample = None
    if args.config != "wsj_mono" or w.total_frames > 40000:
        sample = max(1, int(len(w.seqs) * min(1.0, 20000.0 / max(1, w.total_frames))))
    fps, info = cpu_reference_run(w, steps, args.warmup, sample)
    times = info["times_s"]
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s",
        "n_gpus": world, "steps": steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * float(np.mean(times)), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "B_sampled": info["B"], "frames": info["frames"],
                   "seed": 0},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": info["cores"],
                         "kind": info["kind"],
                         "sample": f"{info['B']} sequences / {info['frames']} frames of "
                                   f"{args.config} seed 0, best of {steps}"},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import torch

    import paper_2005_09824_b200 as P
    from paper_2005_09824_b200 import _backend, synth

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        pg = dist.group.WORLD
    ext = _backend.require_cuda()

    w = synth.make_workload(args.config, seed=rank, batch_size=args.batch)
    batch, nums, den = w.build(P)
    opts = P.FBOptions()
    B, T, D = batch.values.shape
    values = torch.tensor(batch.values, dtype=torch.float32, device=dev)
    lengths = torch.tensor(batch.lengths, dtype=torch.int32, device=dev)
    frames_local = int(batch.lengths.sum())
    grad = torch.empty_like(values)
    ng = P.device_graphs(nums, dev)
    dg = P.device_graphs(den, dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        g, nl, dl, nf, df, totals = P.chain_loss_device(values, lengths, nums, den, opts,
                                                        total_frames=frames_local, grad=grad)
        if pg is not None:
            torch.distributed.all_reduce(totals, group=pg)
        return totals

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    sampler = None
    if rank == 0 and not args.profile:
        sampler = ClockSampler(local)
        sampler.start()
        time.sleep(0.3)
    if pg is not None:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.fill_(i & 0xFF)  # L2 flush, outside the timed events
        starts[i].record(stream)
        step()
        ends[i].record(stream)
    torch.cuda.synchronize()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = float(np.sum(step_ms))
    if pg is not None:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
        fr = torch.tensor([frames_local], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(fr)
        frames_all = int(fr.item())
        torch.distributed.barrier()
    else:
        frames_all = frames_local
    clocks = sampler.stop() if sampler else None
    ms_per_step = total_ms / args.steps
    value = frames_all * args.steps / (total_ms / 1e3)

    # ---- dominant kernel timed alone (no collective), same inputs -----------
    # Fused path (LFMMI_FUSED=1): the single chain launch.  Two-pass path
    # (default): the denominator pass, the step's critical path (the numerator
    # pass runs concurrently on an auxiliary stream; combine + totals ~10 us).
    launches_per_step = int(ext.last_launch_count())
    fused = launches_per_step == 1

    def dominant_launch():
        if fused:
            P.chain_loss_device(values, lengths, nums, den, opts, total_frames=frames_local,
                                grad=grad)
        else:
            P.forward_backward_device(values, lengths, den, opts, posteriors=grad, mode=3,
                                      total_frames=frames_local)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        ev[i][0].record(stream)
        dominant_launch()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    kernel_ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    den_kernel = str(ext.last_den_kernel())  # the kernel dominant_launch() ran

    num_S = [nums.graph(b).num_states for b in range(B)]
    num_I = [nums.graph(b).num_transitions for b in range(B)]
    den_g = den.graph(0)
    A_step = algorithmic_bytes(batch.lengths, D, den_g.num_states, den_g.num_transitions, num_S,
                               num_I)
    # Denominator pass alone: no numerator graphs in its compulsory traffic.
    A = A_step if fused else algorithmic_bytes(batch.lengths, D, den_g.num_states,
                                               den_g.num_transitions, [0], [0])
    peaks = load_json(MEASURED_PEAKS) or {}
    peak = peaks.get("hbm_gbs")
    peak_src = "measured" if peak else "fallback"
    peak = peak or 6650.0
    achieved = A / (kernel_ms / 1e3) / 1e9
    ncu = load_json(NCU_SUMMARY) or {}
    # ncu traffic is recorded for the headline workload only (profiles/ncu_summary.json)
    traffic = None
    if ncu.get("workload", "wsj_mono") == args.config and args.batch is None:
        traffic = ncu.get("chain_dram_bytes_per_launch" if fused else "den_dram_bytes_per_launch")

    # ---- end-to-end through the public API with host buffers ----------------
    e2e = None
    if not args.no_e2e:
        # End to end through the public API: every step copies that step's
        # log-likelihoods + lengths from pinned host memory (on a copy stream,
        # one step ahead, double-buffered) and reads the step's result (the 3
        # totals: objective, frames, failures) back to the host.  The gradient
        # w.r.t. the network output stays on the device for backprop.
        # Inputs in the packed (sum T, D) layout of the device-side batching API
        # (chain_loss_packed): only real frames cross PCIe
        # (9.7 MB per WSJ-mono step instead of the 12.8 MB padded batch).
        lens_np = np.asarray(batch.lengths)
        packed = np.concatenate([np.asarray(batch.values[b, :int(t)], dtype=np.float32)
                                 for b, t in enumerate(lens_np)])
        t_max = int(lens_np.max())
        host_L = [torch.from_numpy(packed).pin_memory() for _ in range(2)]
        host_len = [torch.tensor(lens_np, dtype=torch.int32).pin_memory() for _ in range(2)]
        grad_packed = torch.empty(host_L[0].shape, dtype=torch.float32, device=dev)
        host_tot = torch.empty((args.steps + 8, 3), dtype=torch.float64).pin_memory()
        x_dev = [torch.empty_like(grad_packed) for _ in range(2)]
        l_dev = [torch.empty_like(lengths) for _ in range(2)]
        copy_stream = torch.cuda.Stream(dev)
        d2h_stream = torch.cuda.Stream(dev)  # the totals read-back never blocks the next step
        h2d_done = [torch.cuda.Event() for _ in range(2)]
        used = [torch.cuda.Event() for _ in range(2)]

        def h2d(i):
            j = i & 1
            with torch.cuda.stream(copy_stream):
                copy_stream.wait_event(used[j])  # buffer j free (step i-2 consumed it)
                x_dev[j].copy_(host_L[j], non_blocking=True)
                l_dev[j].copy_(host_len[j], non_blocking=True)
                h2d_done[j].record(copy_stream)

        def compute(i):
            j = i & 1
            stream.wait_event(h2d_done[j])
            g, _, _, _, _, totals = P.chain_loss_packed(x_dev[j], l_dev[j], nums, den, opts,
                                                        max_frames=t_max,
                                                        total_frames=frames_local,
                                                        grad=grad_packed)
            if pg is not None:
                torch.distributed.all_reduce(totals, group=pg)
            used[j].record(stream)
            d2h_stream.wait_event(used[j])
            totals.record_stream(d2h_stream)
            with torch.cuda.stream(d2h_stream):
                host_tot[i].copy_(totals, non_blocking=True)

        def run(n):
            h2d(0)
            for i in range(n):
                if i + 1 < n:
                    h2d(i + 1)
                compute(i)

        run(3)
        torch.cuda.synchronize()
        flush.fill_(0)
        torch.cuda.synchronize()
        t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t_start.record(copy_stream)
        run(args.steps)
        t_end.record(d2h_stream)  # after the last step's totals reached the host buffer
        torch.cuda.synchronize()
        e_ms = t_start.elapsed_time(t_end)
        if pg is not None:
            t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": frames_all * args.steps / (e_ms / 1e3), "unit": "frames/s",
               "h2d_bytes_per_step": int(host_L[0].numel() * 4 + host_len[0].numel() * 4),
               "d2h_bytes_per_step": 3 * 8, "ms_per_step": e_ms / args.steps,
               "how": "chain_loss_packed (ragged sum-T x D input, caller order); "
                      "pinned H2D of each step's inputs on a copy stream (one step ahead, "
                      "double-buffered) + D2H of the step's totals on a read-back stream; "
                      "grad stays on device"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        fps, info = cpu_reference_run(w, 3, 1)
        cpu = {"value": fps, "unit": "frames/s", "cores": info["cores"], "kind": info["kind"],
               "sample": f"full {args.config} batch seed 0 ({info['B']} seqs, {info['frames']} "
                         f"frames), best of 3 after 1 warm-up"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
            "data": "synthetic",
            "config": {"workload": args.config, "S_den": den_g.num_states,
                       "I_den": den_g.num_transitions, "D": D, "B_per_gpu": B,
                       "frames_per_gpu": frames_local, "T_max": T, "seed": "rank",
                       "l2": "flushed (512 MiB write) before every timed step",
                       "parallelism": f"dp{world} (sequence-sharded, scalar all-reduce)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": den_kernel,
                         "algorithmic_bytes_per_launch": A, "launch_ms": kernel_ms,
                         "algorithmic_bytes_per_step": A_step,
                         "peak_source": peak_src},
            "kernel_share_of_step": kernel_ms / ms_per_step,
            "e2e": e2e, "gpu_launches": launches_per_step * args.steps, "cpu_baseline": cpu,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if pg is not None:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
