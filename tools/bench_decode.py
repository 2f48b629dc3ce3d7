#!/usr/bin/env python
"""BASELINE config 4, decode regime: batch 1..64 single text tokens through
the seven Qwen2.5-VL-7B decoder projections with packed W4 / W3 weights.

Reports, per batch size and weight width:
  * the step (seven forwards, replayed as one CUDA graph) in us and tokens/s,
    with the forwards in sequence (step_us) and along the decoder block's
    dataflow, independent projections on parallel streams (step_us_branches:
    q || k || v, o, gate || up, down);
  * the split-GEMM kernels' time (CUDA events around each launch, stage
    profile) and the HBM bandwidth of their weight streaming:
      algorithmic bytes = packed main codes + 4-bit outlier and
      low-rank codes + fp32 scales, per projection;
      streamed bytes = what the kernels actually read for the weights
      (packed main codes + the fp16 auxiliary B operand);
    both divided by the GEMM time, against the measured HBM peak.
One JSON line per (wbits, abits, batch) on stdout.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import workloads as wl  # noqa: E402
import paper_2605_19929_b200 as pkg  # noqa: E402
from paper_2605_19929_b200 import runtime  # noqa: E402


def layer_bytes(sp, lay_k_lr, wbits):
    d_m = sp.d_in - sp.k_text - sp.k_vision
    alg = (d_m * sp.d_out * wbits / 8 + 2 * sp.k_text * sp.d_out * max(wbits, 4) / 8
           + (d_m * sp.r_cws + sp.r_cws * sp.d_out + d_m * sp.r_mac + sp.r_mac * sp.d_out) * 4 / 8
           + (5 * sp.d_out + sp.r_cws + sp.r_mac) * 4)
    ld = (sp.d_in + 15) // 16 * 16
    streamed = sp.d_out * ld / 2 + sp.d_out * lay_k_lr * 2 + sp.d_out * 4 * 3
    return alg, streamed


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", default="1,2,4,8,16,32,64")
    ap.add_argument("--specs", default="4:4,3:3,3:2", help="wbits:abits list")
    ap.add_argument("--iters", type=int, default=50)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    peaks = bench.measured_peaks()
    hbm = peaks.get("hbm_gbs", 6535.4)
    for spec in a.specs.split(","):
        wbits, abits = (int(v) for v in spec.split(":"))
        tags, inputs, layers = bench.build_workload(pkg, 64, abits, wbits)
        gls = [(g, sp, runtime.GpuLayer(layer, dev)) for g, sp, layer in layers]
        for B in (int(b) for b in a.batches.split(",")):
            tg = torch.zeros(B, dtype=torch.uint8, device=dev)  # decode: all text tokens
            xs = {g: bench.make_input_tensor(torch, dev, B, inputs[g], np.zeros(B, np.uint8), 5 + i)
                  for i, g in enumerate(inputs)}
            ws = torch.empty(max(int(gl.layout(B).total_bytes) for _, _, gl in gls),
                             dtype=torch.uint8, device=dev)
            ys = [torch.empty((B, sp.d_out), dtype=torch.float16, device=dev) for _, sp, _ in gls]

            def step(profile=False):
                for (g, sp, gl), y in zip(gls, ys):
                    gl.run(xs[g], tg, y=y, check=False, ws=ws, profile=profile)

            step()
            torch.cuda.synchronize()
            # stage profile (events per stage, eager launches)
            for _, _, gl in gls:
                gl.profile_read()
            for _ in range(a.iters):
                step(profile=True)
            torch.cuda.synchronize()
            gemm_us, alg_b, str_b = {}, 0.0, 0.0
            for g, sp, gl in gls:
                st, calls = gl.profile_read()
                gemm_us[sp.name] = st[2] / calls * 1e3
                al, sb = layer_bytes(sp, int(gl.layout(B).k_lr), wbits)
                alg_b += al
                str_b += sb
            gemm_total_us = sum(gemm_us.values())
            # the whole step as one CUDA graph (launch overheads amortised)
            graph = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                step()
                torch.cuda.synchronize()
                with torch.cuda.graph(graph, stream=s):
                    step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            graph.replay()
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.iters):
                graph.replay()
            e1.record()
            e1.synchronize()
            step_us = e0.elapsed_time(e1) / a.iters * 1e3
            # the decoder block's dataflow: q || k || v, o, gate || up, down
            # (independent projections on their own streams inside one graph;
            # each projection its own workspace)
            wss = [torch.empty(int(gl.layout(B).total_bytes), dtype=torch.uint8, device=dev) for _, _, gl in gls]
            names = [sp.name for _, sp, _ in gls]
            levels = [["q", "k", "v"], ["o"], ["gate", "up"], ["down"]]
            streams = [torch.cuda.Stream() for _ in range(3)]

            def step_branches():
                cur = torch.cuda.current_stream()
                for lvl in levels:
                    ev = torch.cuda.Event()
                    ev.record(cur)
                    done = []
                    for j, nm in enumerate(lvl):
                        i = names.index(nm)
                        g, sp, gl = gls[i]
                        st = streams[j]
                        st.wait_event(ev)
                        with torch.cuda.stream(st):
                            gl.run(xs[g], tg, y=ys[i], check=False, ws=wss[i])
                        e = torch.cuda.Event()
                        e.record(st)
                        done.append(e)
                    for e in done:
                        cur.wait_event(e)

            graph2 = torch.cuda.CUDAGraph()
            s2 = torch.cuda.Stream()
            s2.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s2):
                step_branches()
                torch.cuda.synchronize()
                with torch.cuda.graph(graph2, stream=s2):
                    step_branches()
            torch.cuda.synchronize()
            graph2.replay()
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.iters):
                graph2.replay()
            e1.record()
            e1.synchronize()
            step_br_us = e0.elapsed_time(e1) / a.iters * 1e3
            print(json.dumps({
                "config": "config4 decode: Qwen2.5-VL-7B q,k,v,o,gate,up,down, all-text tokens",
                "wbits": wbits, "abits": abits, "batch": B,
                "step_us": step_us, "tokens_per_s": B / (step_us * 1e-6),
                "step_us_branches": step_br_us, "tokens_per_s_branches": B / (step_br_us * 1e-6),
                "gemm_us_total": gemm_total_us, "gemm_us": gemm_us,
                "weight_bytes_algorithmic": alg_b, "weight_bytes_streamed": str_b,
                "hbm_gbs_algorithmic": alg_b / (gemm_total_us * 1e-6) / 1e9,
                "hbm_gbs_streamed": str_b / (gemm_total_us * 1e-6) / 1e9,
                "hbm_peak_gbs": hbm,
                "frac_streamed": str_b / (gemm_total_us * 1e-6) / 1e9 / hbm,
            }), flush=True)


if __name__ == "__main__":
    main()
