"""Shared pieces of the bench.py workloads: peaks, clocks, host description,
process-group setup, CUDA-event timing."""

from __future__ import annotations

import json
import os
import statistics
import subprocess
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
HBM_PEAK_FALLBACK = 6650.0  # GB/s, B200_PROFILING.md fallback


def peaks() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_PEAK_FALLBACK, "fallback (B200_PROFILING.md)"


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def host_cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def dist_env() -> tuple[int, int, int]:
    """(world, rank, local_rank) from the torchrun environment."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # TDP_ONE_GPU=1 (+ TDP_DIST_BACKEND=gloo) runs several ranks on cuda:0 to
    # exercise the multi-rank code path on a single-GPU host
    if os.environ.get("TDP_ONE_GPU") == "1":
        local = 0
    return world, rank, local


def init_dist(world: int, local: int):
    """Process group over NCCL (one GPU per rank); None for one rank unless
    TDP_FORCE_DIST=1 asks for a real one-rank NCCL communicator."""
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1 or os.environ.get("TDP_FORCE_DIST") == "1":
        backend = os.environ.get("TDP_DIST_BACKEND", "nccl")
        if not dist.is_initialized():
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            else:
                dist.init_process_group(backend)
        return dist.group.WORLD
    return None


def max_over_ranks(vals: list[float], group) -> list[float]:
    import torch
    import torch.distributed as dist

    if group is None:
        return vals
    t = torch.tensor(vals, dtype=torch.float64, device="cuda")
    if dist.get_backend(group) == "gloo":
        t = t.cpu()
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return [float(x) for x in t.tolist()]


def sum_over_ranks(v: int, group) -> int:
    import torch
    import torch.distributed as dist

    if group is None:
        return v
    t = torch.tensor([v], dtype=torch.int64, device="cuda")
    if dist.get_backend(group) == "gloo":
        t = t.cpu()
    dist.all_reduce(t, group=group)
    return int(t.item())


def barrier(group) -> None:
    import torch.distributed as dist

    if group is not None:
        dist.barrier(group=group)


def timed(fn, steps: int, group=None) -> float:
    """ms per call of ``fn`` over ``steps`` calls: CUDA events on the current
    stream, barrier + synchronize on both sides, max over ranks."""
    import torch

    barrier(group)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(steps):
        fn()
    t1.record()
    torch.cuda.synchronize()
    barrier(group)
    return max_over_ranks([t0.elapsed_time(t1) / steps], group)[0]


def sustain(fn, seconds: float = 1.5) -> int:
    """Call ``fn`` back to back for ``seconds`` of wall time (clock sampling
    needs a loaded GPU for longer than nvidia-smi's sampling period)."""
    import torch

    n = 0
    w0 = time.perf_counter()
    while time.perf_counter() - w0 < seconds:
        for _ in range(8):
            fn()
        n += 8
        torch.cuda.synchronize()
    return n


class ClockSampler:
    """nvidia-smi clock / throttle-reason samples while ``active``."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, device_index: int = 0):
        import torch

        uuid = str(torch.cuda.get_device_properties(device_index).uuid)
        gpu_id = uuid if uuid.startswith("GPU-") else "GPU-" + uuid
        self.samples: list[list[str]] = []
        self.proc = None
        self.active = False
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", gpu_id, f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            return
        self._first = threading.Event()
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        self._first.wait(timeout=5.0)

    def _read(self):
        for line in self.proc.stdout:
            self._first.set()
            if self.active:
                self.samples.append([x.strip() for x in line.split(",")])

    def stop(self) -> dict:
        self.active = False
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "note": "nvidia-smi unavailable"}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()]
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}
