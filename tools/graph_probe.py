"""Probe: the C4 step (compact keys) replayed from a CUDA graph vs launched
eagerly; checks the graph's record and histogram equal the eager ones."""
import json
import math
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1511_07983_b200 import workloads as W  # noqa: E402
from paper_1511_07983_b200.sweep import Sweeper  # noqa: E402

gpu, ks = W.config("C4")
sw = Sweeper(gpu, device=0, compact_keys=True)
sw.set_kernels(ks)
_, idx = sw.heuristic()
s = torch.cuda.Stream()
out = {}
with torch.cuda.stream(s):
    for _ in range(3):
        sw.step_device(idx, s)
torch.cuda.synchronize()
ref = torch.cat([sw.record, sw.hist]).clone()


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


with torch.cuda.stream(s):
    out["eager_ms"] = timeit(lambda: sw.step_device(idx, s))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        sw.step_device(idx, s)
    g.replay()
    torch.cuda.synchronize()
    out["graph_ms"] = timeit(g.replay)
torch.cuda.synchronize()
out["graph_equal"] = bool(torch.equal(torch.cat([sw.record, sw.hist]), ref))
print(json.dumps(out))
