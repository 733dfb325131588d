"""Single-shot latency at C3 from pinned host memory: (a) plain H2D of the 32-bit CSR then the
pipeline; (b) the compact u16 wire format through ingest.upload_qc (chunked H2D, per-chunk decode
and QC while later chunks are in flight) then the rest of the pipeline.  Prints one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_13928_b200 import ingest, pipeline, synth  # noqa: E402
from paper_2605_13928_b200.pp import DeviceCSR  # noqa: E402

spec = synth.Spec(1_000_000, 25_000, seed=0)
X = synth.generate(spec)
mt = synth.mt_mask(spec)
p = pipeline.Params()
H32 = ingest.HostCSR.from_device(X)
H16 = ingest.HostCSR.from_device(X.to_u16())
del X
torch.cuda.empty_cache()
out = {}
for rep in range(2):
    e0, e1, e2 = (torch.cuda.Event(True) for _ in range(3))
    e0.record()
    Xd = DeviceCSR(H32.indptr.to("cuda", non_blocking=True), H32.indices.to("cuda", non_blocking=True),
                   H32.data.to("cuda", non_blocking=True), H32.n_cols)
    e1.record()
    r = pipeline.run(Xd, mt, p, timing=False)
    e2.record()
    torch.cuda.synchronize()
    out["plain_f32"] = {"h2d_ms": round(e0.elapsed_time(e1), 1), "total_ms": round(e0.elapsed_time(e2), 1)}
    del Xd, r
    torch.cuda.empty_cache()
    e0, e1, e2 = (torch.cuda.Event(True) for _ in range(3))
    e0.record()
    Xd, qc = ingest.upload_qc(H16, mt, chunk_rows=1 << 16)
    e1.record()
    r = pipeline.run(Xd, mt, p, timing=False, qc=qc)
    e2.record()
    torch.cuda.synchronize()
    out["upload_qc_u16"] = {"upload_decode_qc_ms": round(e0.elapsed_time(e1), 1), "total_ms": round(e0.elapsed_time(e2), 1)}
    del Xd, r, qc
    torch.cuda.empty_cache()
print(json.dumps(out))
