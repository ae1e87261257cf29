"""cmvg_create wall time at C2 (n = 2^24): device build (default) vs host
build (CMVG_HOST_BUILD=1); dev tool for the GPU box."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1708_07271_b200 as P

nlog = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g = P.CsrGraph.copy_model(1 << nlog, 20.0, 0.7, 0.8, seed=0x170807271 + 2)
s = P.BvStream.encode(g, P.BvParams())
out = {}
import torch
torch.cuda.init()
for mode in ("device", "host", "device"):
    if mode == "host":
        os.environ["CMVG_HOST_BUILD"] = "1"
    else:
        os.environ.pop("CMVG_HOST_BUILD", None)
    t = time.time()
    dg = P.BvGraph(s)
    out[mode] = time.time() - t
    w, b, dev = dg.bvf_export()
    out[mode + "_device_built"] = dev
    out[mode + "_words"] = int(len(w))
    del dg
print(json.dumps(out))
