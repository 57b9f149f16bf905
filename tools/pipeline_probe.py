"""Probe: two C4 steps in flight (two contexts = two sets of memo tables and
key buffers, one stream each), so step i+1's latency-bound pass 1 overlaps
step i's HBM-bound key stream.  Prints ms/step for 1 and 2 streams, with and
without a high-priority stream for the pass-1-heavy side."""
import json
import math
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1511_07983_b200 import workloads as W  # noqa: E402
from paper_1511_07983_b200.sweep import Sweeper  # noqa: E402

gpu, ks = W.config("C4")
N = math.factorial(12)
out = {}
for mode in ("one", "two", "two_prio"):
    nsw = 1 if mode == "one" else 2
    sws = [Sweeper(gpu, device=0, compact_keys=True) for _ in range(nsw)]
    lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
    streams = [torch.cuda.Stream(priority=(-1 if (mode == "two_prio") else 0)) for _ in range(nsw)]
    for s in sws:
        s.set_kernels(ks)
    _, idx = sws[0].heuristic()
    main = torch.cuda.current_stream()
    for rep in range(2):
        K = 20
        for i in range(4):
            with torch.cuda.stream(streams[i % nsw]):
                sws[i % nsw].step_device(idx, streams[i % nsw])
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        for s in streams:
            s.wait_stream(main)
        for i in range(K):
            st = streams[i % nsw]
            with torch.cuda.stream(st):
                sws[i % nsw].step_device(idx, st)
        for s in streams:
            main.wait_stream(s)
        b.record(main)
        torch.cuda.synchronize()
        out[mode] = a.elapsed_time(b) / K
    for s in sws:
        assert int(s.hist.sum().item()) == N
    del sws
    torch.cuda.empty_cache()
print(json.dumps(out))
