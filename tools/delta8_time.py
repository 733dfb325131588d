"""Device time of scb_csr_delta8_decode on the C3 matrix (byte-delta wire -> int32/float32 CSR)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_13928_b200 import synth
from paper_2605_13928_b200.pp import DeltaCSR, DeviceCSR
spec = synth.Spec(1_000_000, 25_000, seed=0)
X = synth.generate(spec)
D = DeltaCSR.from_csr(X)
out = DeviceCSR(X.indptr, torch.empty_like(X.indices), torch.empty_like(X.data), X.n_cols)
ms = []
for _ in range(6):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(); D.to_f32(out=out); b.record(); torch.cuda.synchronize()
    ms.append(round(a.elapsed_time(b), 3))
ok = torch.equal(out.indices, X.indices) and torch.equal(out.data, X.data)
gb = (2 * X.nnz + 8 * (X.n_rows + 1) + 8 * X.nnz) / 1e9
print(f"[delta8] nnz {X.nnz} ms {ms} bit_identical {ok} algorithmic {gb:.2f} GB -> {gb / min(ms[1:]) * 1e3:.0f} GB/s at best")
