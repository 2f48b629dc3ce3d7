#!/usr/bin/env python
"""SplitQ split-linear bench (driver contract: one JSON line on rank 0).

Workload (BASELINE.json config 3, the metric's config): the seven
Qwen2.5-VL-7B decoder projections (q, k, v, o, gate, up, down) at W4A4
(activations asymmetric per token, weights symmetric per channel, CWS + MAC
on, 32 + 32 outlier channels per layer input) over a batch of 8 samples x
8192 tokens (1280 vision tokens in contiguous spans + 6912 text tokens per
sample). One "step" = all seven projections over the whole batch; tokens
are sharded across ranks (strong scaling), with no collective on the path.

  value  tokens/s of the whole job (all ranks), device time, inputs resident in HBM
  e2e    same metric through the public API with host (pinned) inputs and outputs,
         H2D + D2H copies inside the timed region
  roofline  split GEMM kernel vs the measured dense INT8 tensor peak

``--impl reference`` times the CPU oracle port (oracle/splitq_oracle.py, a
restatement of the reference numpy path) on the same config; the reference
package itself is pure Python and is not installed on the GPU box.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as wl  # noqa: E402

SAMPLES, SEQ, VISION_PER_SAMPLE = 8, 8192, 1280
METRIC = "W4A4 split-linear tokens/sec (7B shapes) at 1/2/4/8 B200; % INT8 TC peak"
DATASHEET_INT8_TOPS = 4500.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--tokens", type=int, default=SAMPLES * SEQ, help="global tokens per step")
    ap.add_argument("--abits", type=int, default=4)
    ap.add_argument("--wbits", type=int, default=4)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-tokens", type=int, default=256)
    ap.add_argument("--out-dtype", default="float16", choices=["float16", "bfloat16", "float32"])
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def measured_peaks():
    peaks = {}
    for path in (os.path.join(ROOT, "MEASURED_PEAKS.json"),):
        try:
            with open(path) as fh:
                peaks.update(json.load(fh))
        except (OSError, ValueError):
            pass
    try:
        with open(os.path.join(ROOT, "profiles", "int8_peak.json")) as fh:
            peaks["int8"] = json.load(fh)
    except (OSError, ValueError):
        pass
    return peaks


# ------------------------------------------------------------------ workload

def build_workload(pkg, tokens, abits, wbits, seed=0):
    """Layer inputs (one per distinct projection input) and the 7 layers."""
    rng = np.random.default_rng(seed)
    shape = wl.QWEN_7B
    specs = wl.model_specs(shape, abits=abits, wbits=wbits)
    n_samples = max(1, tokens // SEQ)
    tags = np.concatenate([wl.tags_with_spans(rng, SEQ, VISION_PER_SAMPLE)
                           for _ in range(n_samples)])[:tokens]
    if tags.shape[0] < tokens:  # non-multiple of SEQ
        tags = np.concatenate([tags, wl.tags_with_spans(rng, tokens - tags.shape[0],
                                                        (tokens - tags.shape[0]) * 5 // 32)])
    inputs = {}
    groups = {"qkv": ("q", "k", "v"), "o": ("o",), "gu": ("gate", "up"), "down": ("down",)}
    layers = []
    for gname, members in groups.items():
        sp0 = next(s for s in specs if s.name == members[0])
        c_t, c_v = wl.outlier_sets(rng, sp0.d_in, sp0.k_text)
        inputs[gname] = dict(c_t=c_t, c_v=c_v, d_in=sp0.d_in)
        # per-channel max |X| of this input (calibration statistic for the transforms)
        scales_t = rng.uniform(30, 100, len(c_t))
        scales_v = rng.uniform(30, 100, len(c_v))
        inputs[gname].update(scales_t=scales_t, scales_v=scales_v)
        col_max = np.full(sp0.d_in, 4.5)
        col_max[c_t] = 4.5 * scales_t
        col_max[c_v] = 4.5 * scales_v
        for m in members:
            sp = next(s for s in specs if s.name == m)
            layers.append((gname, sp, wl.build_split_layer(pkg, rng, sp, col_max, c_t, c_v)))
    return tags, inputs, layers


def make_input_tensor(torch, dev, tokens, spec_in, tags, seed):
    """N(0,1) fp16 activations with the planted outlier scales, made on device."""
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    x = torch.randn((tokens, spec_in["d_in"]), generator=g, device=dev, dtype=torch.float32)
    t = torch.from_numpy(tags).to(dev)
    text = (t == 0).unsqueeze(1)
    ct = torch.from_numpy(spec_in["c_t"]).to(dev)
    cv = torch.from_numpy(spec_in["c_v"]).to(dev)
    st = torch.from_numpy(spec_in["scales_t"]).to(dev, torch.float32)
    sv = torch.from_numpy(spec_in["scales_v"]).to(dev, torch.float32)
    x[:, ct] = torch.where(text, x[:, ct] * st, x[:, ct])
    x[:, cv] = torch.where(~text, x[:, cv] * sv, x[:, cv])
    return x.to(torch.float16)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sms, maxes, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            f = [c.strip() for c in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm, mx = float(f[0]), float(f[1])
            except ValueError:
                continue
            sms.append(sm)
            maxes.append(mx)
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sms:
            return None
        loaded = [s for s in sms if s > 0.5 * max(sms)] or sms
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(maxes),
                "reasons": sorted(reasons), "samples": len(sms)}


# ------------------------------------------------------------------ arms

def run_ours(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", torch.cuda.current_device())

    import paper_2605_19929_b200 as pkg
    from paper_2605_19929_b200 import _lib, runtime

    lib = _lib.load()
    global_tokens = args.tokens
    tokens = global_tokens // world  # strong scaling: the batch is sharded by samples / rows
    tags_all, inputs, layers = build_workload(pkg, global_tokens, args.abits, args.wbits)
    tags_np = np.ascontiguousarray(tags_all[rank * tokens:(rank + 1) * tokens])
    tags = torch.from_numpy(tags_np).to(dev)
    xs = {g: make_input_tensor(torch, dev, tokens, inputs[g], tags_np, 1000 + 17 * rank + i)
          for i, g in enumerate(inputs)}
    packed = [(g, sp, runtime.GpuLayer(layer, dev)) for g, sp, layer in layers]
    ws_bytes = max(int(gl.layout(tokens).total_bytes) for _, _, gl in packed)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    out_dt = getattr(torch, args.out_dtype)
    ys = [torch.empty((tokens, sp.d_out), dtype=out_dt, device=dev) for _, sp, _ in packed]
    stream = torch.cuda.current_stream()

    def step(profile=False):
        for (g, sp, gl), y in zip(packed, ys):
            gl.run(xs[g], tags, y=y, check=False, ws=ws, profile=profile)

    # correctness gate before timing: device error word clear
    step()
    st = np.zeros(1, np.int32)
    import ctypes as C
    stv = C.c_int32()
    _lib.check(lib.splitq_read_status(C.c_void_p(ws.data_ptr()), C.c_void_p(stream.cuda_stream),
                                      C.byref(stv)))
    for _ in range(args.warmup):
        step()
    for _, _, gl in packed:
        gl.profile_read()  # drop warm-up events
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(dev.index)
    clocks.start()
    time.sleep(0.3)
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    start.record(stream)
    for _ in range(args.steps):
        step(profile=True)
    end.record(stream)
    end.synchronize()
    ms = start.elapsed_time(end)
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps

    # stage split and the roofline of the split GEMM (algorithmic int8 ops per launch)
    stage = np.zeros(3)
    gemm_ops = 0.0
    launches = 0
    per_layer = {}
    for g, sp, gl in packed:
        st_ms, calls = gl.profile_read()
        stage += np.array(st_ms)
        gemm_ops += 2.0 * tokens * sp.d_in * sp.d_out * calls
        launches += calls * (2 + (1 if sp.r_cws else 0) + (1 if sp.r_mac else 0) + 1)
        per_layer[sp.name] = {"quant_ms": st_ms[0] / max(calls, 1), "lr1_ms": st_ms[1] / max(calls, 1),
                              "gemm_ms": st_ms[2] / max(calls, 1),
                              "gemm_tops": 2.0 * tokens * sp.d_in * sp.d_out / (st_ms[2] / max(calls, 1)) / 1e9}
    gemm_ms_total = stage[2]
    achieved_tops = gemm_ops / (gemm_ms_total * 1e-3) / 1e12
    peaks = measured_peaks()
    int8 = peaks.get("int8") or {}
    peak_tops = int8.get("int8_tops_sustained") or int8.get("int8_tops")
    peak_src = "measured cuBLASLt int8 8192^3 (profiles/int8_peak.json, sustained)"
    if not peak_tops:
        peak_tops = DATASHEET_INT8_TOPS
        peak_src = "datasheet dense INT8 (no measured INT8 entry)"

    value = global_tokens * args.steps / (ms * 1e-3)
    result = {
        "metric": METRIC,
        "value": value,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "int8 (W4A4 codes on tcgen05 kind::i8, int32 accumulate)",
        "data": "synthetic (seeded N(0,1) fp16 activations with x30-x100 outlier channels; "
                "random-init weights and low-rank factors)",
        "config": {
            "workload": "config3: Qwen2.5-VL-7B decoder projections q,k,v,o,gate,up,down; W4A4 "
                        "(A asym per-token, W sym per-channel), CWS+MAC on, K_t=K_v=32",
            "global_tokens": global_tokens, "tokens_per_gpu": tokens,
            "samples": SAMPLES, "seq_len": SEQ, "vision_tokens_per_sample": VISION_PER_SAMPLE,
            "parallelism": f"token-sharded replicas x{world} (no collective on the path)",
            "out_dtype": args.out_dtype, "abits": args.abits, "wbits": args.wbits,
            "l2": "inputs larger than L2 (each projection input >= 470 MB at N=1)",
        },
        "stage_ms_per_step": {"quantize": stage[0] / args.steps, "lowrank_first_stage": stage[1] / args.steps,
                              "split_gemm": stage[2] / args.steps},
        "per_projection": per_layer,
        "roofline": {
            "bound": "tensor",
            "kernel": "splitq_gemm_kernel (split GEMM)",
            "achieved": achieved_tops,
            "peak": peak_tops,
            "unit": "TFLOP/s",
            "frac": achieved_tops / peak_tops,
            "peak_source": peak_src,
            "frac_of_datasheet_4500": achieved_tops / DATASHEET_INT8_TOPS,
            "traffic": None,
            "algorithmic_ops": "2*T*D_in*D_out per projection (dense-equivalent, SURVEY 8(d))",
        },
        "gpu_launches": launches,
        "clocks": clk,
    }

    if not args.no_e2e:
        result["e2e"] = run_e2e(args, torch, dev, packed, xs, tags_np, ws, out_dt, global_tokens, world)
    if world > 1:
        dist.barrier()
    if rank == 0:
        if not args.no_cpu_baseline and world == 1:
            result["cpu_baseline"] = cpu_baseline(layers, inputs, tags_all, args.cpu_sample_tokens)
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, torch, dev, packed, xs, tags_np, ws, out_dt, global_tokens, world):
    """Public-API path with host buffers: pinned inputs -> device, 7 forwards,
    outputs -> pinned host, every step inside the timed region."""
    import torch.distributed as dist

    host_x = {g: x.cpu().pin_memory() for g, x in xs.items()}
    host_tags = torch.from_numpy(tags_np).pin_memory()
    dev_x = {g: torch.empty_like(x) for g, x in xs.items()}
    dev_tags = torch.empty(host_tags.shape, dtype=torch.uint8, device=dev)
    host_y = [torch.empty((x.shape[0], sp.d_out), dtype=out_dt).pin_memory()
              for (g, sp, _), x in zip(packed, [xs[g] for g, _, _ in packed])]
    dev_y = [torch.empty(h.shape, dtype=out_dt, device=dev) for h in host_y]
    h2d = sum(x.numel() * x.element_size() for x in host_x.values()) + host_tags.numel()
    d2h = sum(h.numel() * h.element_size() for h in host_y)

    def step():
        for g in host_x:
            dev_x[g].copy_(host_x[g], non_blocking=True)
        dev_tags.copy_(host_tags, non_blocking=True)
        for (g, sp, gl), y in zip(packed, dev_y):
            gl.run(dev_x[g], dev_tags, y=y, check=False, ws=ws)
        for y, h in zip(dev_y, host_y):
            h.copy_(y, non_blocking=True)

    steps = max(2, min(args.steps, 5))
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        step()
    e.record()
    e.synchronize()
    ms = s.elapsed_time(e)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"value": global_tokens * steps / (ms * 1e-3), "unit": "tokens/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": steps,
            "ms_per_step": ms / steps, "api": "GpuLayer.run (C-ABI splitq_forward) per projection"}


def cpu_baseline(layers, inputs, tags_all, sample_tokens, seed=7):
    """The CPU oracle port (numpy fp64 restatement of the reference forward,
    oracle/splitq_oracle.py) over a bounded sample of the same workload."""
    from oracle import splitq_oracle as orc

    rng = np.random.default_rng(seed)
    tags = tags_all[:sample_tokens]
    total = 0.0
    for g, sp, layer in layers:
        spec_in = inputs[g]
        x = rng.standard_normal((sample_tokens, sp.d_in))
        x[np.ix_(tags == 0, spec_in["c_t"])] *= spec_in["scales_t"]
        x[np.ix_(tags == 1, spec_in["c_v"])] *= spec_in["scales_v"]
        x = x.astype(np.float16).astype(np.float64)
        L = orc.from_reference_layer(layer)
        t0 = time.perf_counter()
        orc.forward(L, x, tags)
        total += time.perf_counter() - t0
    return {"value": sample_tokens / total, "unit": "tokens/s", "cores": os.cpu_count(),
            "kind": "port",
            "sample": f"{sample_tokens} tokens through all 7 projections (same layers, fp64 numpy; "
                      f"includes per-call weight re-quantization like the reference; BLAS threads = "
                      f"{os.cpu_count()}, elementwise single-threaded)",
            "seconds": total}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import paper_2605_19929_b200 as pkg

    tokens_sample = args.cpu_sample_tokens
    tags_all, inputs, layers = build_workload(pkg, max(args.tokens // max(world, 1), SEQ),
                                              args.abits, args.wbits)
    for _ in range(args.warmup and 1):
        cpu_baseline(layers, inputs, tags_all, 32)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vals.append(cpu_baseline(layers, inputs, tags_all, tokens_sample))
    wall = time.perf_counter() - t0
    v = float(np.median([b["value"] for b in vals]))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64 (numpy fake-quantization, as the reference)", "data": "synthetic",
        "config": {"workload": "config3: Qwen2.5-VL-7B decoder projections q,k,v,o,gate,up,down; "
                               "W4A4, CWS+MAC on, K_t=K_v=32",
                   "sample_tokens_per_step": tokens_sample},
        "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
                         "sample": vals[0]["sample"]},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
