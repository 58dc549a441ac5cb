"""Image query (BASELINE config 5): group-by-count over synthetic 28x28
images with a random-init CNN UDF predicate, counts fed to an LLP loss."""

from __future__ import annotations

import json

from .common import ClockSampler


def run(args):
    """Image query (SURVEY config 5): GROUP BY the PE output of a random-init CNN
    UDF over 1e7 synthetic 28x28 images, counts fed to an MSE loss, trained
    with tq.train().  The CNN runs in cuDNN (library code, float32 without
    TF32); the framework's own kernels are the softmax / soft group-by count
    forward and backward.  Their share of the step is taken from one
    torch.profiler pass after the timed region (diagnostic only)."""
    import numpy as np
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_2211_02753_b200 as tq
    from paper_2211_02753_b200 import _native
    from paper_2211_02753_b200.models import TorchModel
    from paper_2211_02753_b200.training import TrainConfig

    torch.cuda.set_device(0)
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.benchmark = True
    n, k = args.image_rows, args.image_classes
    g = torch.Generator(device="cuda").manual_seed(3)
    images = torch.rand(n, 28, 28, generator=g, device="cuda", dtype=torch.float32)
    torch.manual_seed(0)
    net = torch.nn.Sequential(
        torch.nn.Unflatten(1, (1, 28)),
        torch.nn.Conv2d(1, 8, 3), torch.nn.ReLU(), torch.nn.MaxPool2d(2),
        torch.nn.Conv2d(8, 16, 3), torch.nn.ReLU(), torch.nn.MaxPool2d(2),
        torch.nn.Flatten(), torch.nn.Linear(400, k)).cuda()
    chunk = 1 << 18
    model = TorchModel(net, "cnn", chunk_rows=chunk)
    reg = tq.UdfRegistry()
    reg.register(tq.classifier_tvf("cnn", model, k, "Pred"))
    cat = tq.Catalog()
    X = tq.Tensor(images)
    cat.register_tensor(X, "imgs")
    q = tq.compile_plan(tq.lower(tq.bind(tq.parse(
        "SELECT Pred, COUNT(*) FROM cnn(imgs) GROUP BY Pred"), cat, reg)),
        tq.CompileConfig(trainable=True), reg)
    target = torch.full((k,), n / k, dtype=torch.float32, device="cuda")
    target[0] *= 1.5
    target[1] *= 0.5
    batches = [("imgs", X, tq.Tensor(target))]
    losses = tq.train(q, cat, batches, TrainConfig(iterations=max(args.warmup, 3), lr=0.01))
    torch.cuda.synchronize()
    launches0 = _native.launch_count()
    steps = max(1, min(args.steps, 5))
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(0)
    sampler.active = True
    t0.record()
    losses += tq.train(q, cat, batches, TrainConfig(iterations=steps, lr=0.01))
    t1.record()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ms = t0.elapsed_time(t1) / steps
    launches = _native.launch_count() - launches0
    # diagnostic: share of one step's device time in this framework's kernels
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        tq.train(q, cat, batches, TrainConfig(iterations=1, lr=0.01))
        torch.cuda.synchronize()
    ours = total = 0.0
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            t = e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
            total += t
            if "tdp::" in e.name:
                ours += t
    line = {
        "metric": "Image query step latency (SURVEY config 5)", "value": ms, "unit": "ms/step",
        "higher_is_better": False, "n_gpus": 1, "steps": steps, "warmup": max(args.warmup, 3),
        "images_per_s": n / (ms / 1e3), "dtype": "f32 (cuDNN convolutions without TF32)",
        "data": "synthetic images U[0,1) (seed 3), random-init CNN",
        "config": {"workload": "SELECT Pred, COUNT(*) FROM cnn(imgs) GROUP BY Pred (trainable), "
                               "CNN conv(1-8,3)+ReLU+pool2 -> conv(8-16,3)+ReLU+pool2 -> FC(400,k) "
                               "-> pe_encode, MSE, Adam",
                   "images": n, "classes": k, "chunk_rows": chunk,
                   "step": "one iteration of tq.train(); CNN activations checkpointed per chunk"},
        "gpu_launches": launches, "clocks": clocks,
        "framework_kernel_share": ours / total if total else None,
        "framework_kernel_ms": ours / 1e3,
        "losses": losses[:2] + losses[-2:],
    }
    print(json.dumps(line), flush=True)
