"""C4: the paper's subsampling sweep on one B200 -- the first n cells of the C3
spec for n = 100k..1M, full QC->kNN pipeline, one CudaMon-style session per n (NVML samples +
step markers, paper_2605_13928_b200.trace) plus CUDA-event per-step times and peak allocator
memory.  Output: <out>/n<cells>/ session dirs and <out>/summary.json.  Analyse with
tools/analyze_c4.py (which uses the reference's own gputrace parser where it is available).

usage: python tools/sweep_c4.py [out_dir] [step_cells] [max_cells]
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_13928_b200 import pipeline, synth, trace  # noqa: E402


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c4"
    step = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 1_000_000
    os.makedirs(out, exist_ok=True)
    G = 25_000
    full = synth.Spec(top, G, seed=0)
    mt = synth.mt_mask(full)
    rows = []
    for n in range(step, top + 1, step):
        X = synth.generate_rows(full, 0, n)  # the first n cells of the C3 matrix
        pipeline.run(X, mt, pipeline.Params(), timing=False)  # warm-up (kernel load, workspaces)
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        sdir = os.path.join(out, f"n{n}")
        h = trace.start(trace.SamplerConfig(sdir, period=0.01, device_index=torch.cuda.current_device()))
        time.sleep(0.05)
        res = pipeline.run(X, mt, pipeline.Params(), mark=h.mark, timing=True)
        torch.cuda.synchronize()
        h.mark("end")
        time.sleep(0.05)
        h.stop()
        peak = torch.cuda.max_memory_allocated()
        trace.write_device_steps(sdir, res.step_ms, {"cells": n, "genes": G, "nnz": X.nnz,
                                                     "peak_allocated_bytes": peak})
        rows.append({"cells": n, "nnz": int(X.nnz), "step_ms": {k: round(v, 3) for k, v in res.step_ms.items()},
                     "total_ms": round(sum(res.step_ms.values()), 3), "peak_allocated_bytes": int(peak)})
        print(json.dumps(rows[-1]), flush=True)
        del X, res
        torch.cuda.empty_cache()
    with open(os.path.join(out, "summary.json"), "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
