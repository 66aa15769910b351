"""C4 end-to-end (pinned host inputs -> streamed backward -> host results) for a few
chunk / block0 choices (dev aid; bench.py's e2e uses 16 chunks, block0 256)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1907_10134_b200.stream import StreamedRnnBackward  # noqa: E402

T, B, H, I = bench.C4["T"], bench.C4["B"], bench.C4["H"], bench.C4["I"]
x, h, p, g = bench.c4_inputs_gpu(0, torch.device("cuda"))
hp, xp = h.cpu().pin_memory(), x.cpu().pin_memory()
del h, x
torch.cuda.empty_cache()
Wp, gp = torch.from_numpy(p["W_hh"]).pin_memory(), torch.from_numpy(g).pin_memory()
outs = [torch.empty(s, pin_memory=True) for s in ((H, I), (H, H), (H,), (B, H))]
for chunks, b0, tail in [(16, 256, 0), (16, 128, 0), (32, 256, 0), (16, 512, 0), (8, 256, 0), (16, 256, 1)]:
    sb = StreamedRnnBackward(T, B, H, I, chunks=chunks, block0=b0, block=bench.C4_BLOCK, tail=tail)
    sb.run(hp, xp, Wp, gp, out_host=outs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        sb.run(hp, xp, Wp, gp, out_host=outs)
    e1.record()
    torch.cuda.synchronize()
    print(f"chunks {chunks} block0 {b0} tail {tail}: e2e {e0.elapsed_time(e1) / 3:.2f} ms", flush=True)
    del sb
    torch.cuda.empty_cache()
