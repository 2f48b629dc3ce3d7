"""Debug counters of the K1 fallback paths (build with -DKW_DEBUG)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2605_19929_b200 as pkg
from paper_2605_19929_b200 import runtime
T = 8192
ABITS = int(sys.argv[1]) if len(sys.argv) > 1 else 4
tags, inputs, layers = bench.build_workload(pkg, T, ABITS, 4)
dev = torch.device("cuda", 0)
tg = torch.from_numpy(tags).to(dev)
for g, sp, layer in layers:
    x = bench.make_input_tensor(torch, dev, T, inputs[g], tags, 1000)
    gl = runtime.GpuLayer(layer, dev)
    ws = gl.workspace(T)
    y = gl.run(x, tg, ws=ws, check=False, out_dtype=torch.float16)
    torch.cuda.synchronize()
    st = ws[:32].cpu().numpy().view(np.int32)
    print(f"A{ABITS}", sp.name, "flagged chunks E:", st[1], "G:", st[3], "rows allx:", st[2] & 0xFFFF,
          "allg:", st[2] >> 16, "unsafe main:", st[5], "unsafe mac:", st[6], "text rows:", int((tags == 0).sum()))
