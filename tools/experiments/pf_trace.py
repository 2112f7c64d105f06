"""Per-tile timeline of CTA 0 of the prefill kernel (C3 workload), from a trace build
(tools/ab/trace/libmvb200.so: clock64 stamps in g_pf_trace).  Writes gpurun_out/pf_trace.npy."""
import ctypes
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)


def main():
    import paper_2506_09991_b200 as mv
    from tools.workloads import nested_16k
    toks = nested_16k()
    n, hq, hkv = len(toks), 40, 8
    g = torch.Generator(device="cuda").manual_seed(0)
    rnd = lambda *s: (torch.rand(*s, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)  # noqa: E731
    q, k, v = rnd(n, hq, 128), rnd(n, hkv, 128), rnd(n, hkv, 128)
    spec = mv.dag.build_visibility(toks)
    out = torch.empty_like(q)
    ws = torch.empty(mv.lib.mv_prefill_workspace_size(n, hq, hkv), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        mv.attention.prefill(q, k, v, spec.positions, spec.excl, out=out, workspace=ws)
    torch.cuda.synchronize()
    buf = np.zeros((12, 8192), np.int64)
    mv.lib.mv_pf_trace_read.argtypes = [ctypes.c_void_p]
    assert mv.lib.mv_pf_trace_read(buf.ctypes.data) == 0
    np.save(os.path.join(REPO, "gpurun_out", "pf_trace.npy"), buf)
    print("ok")


if __name__ == "__main__":
    main()
