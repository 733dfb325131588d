# pinned H2D bandwidth: one stream, two streams, and overlapped with a compute-heavy kernel
import torch, time
n = 1 << 30  # 4 GiB of float32
h = torch.empty(n, dtype=torch.float32).pin_memory()
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float32, device="cuda")
for rep in range(3):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(); d.copy_(h, non_blocking=True); b.record(); torch.cuda.synchronize()
    print(f"1 stream: {4 * n / a.elapsed_time(b) / 1e6:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
half = n // 2
a, b = torch.cuda.Event(True), torch.cuda.Event(True)
a.record()
with torch.cuda.stream(s1): d[:half].copy_(h[:half], non_blocking=True)
with torch.cuda.stream(s2): d[half:].copy_(h[half:], non_blocking=True)
torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
b.record(); torch.cuda.synchronize()
print(f"2 streams: {4 * n / a.elapsed_time(b) / 1e6:.1f} GB/s")
x = torch.randn(8192, 8192, device="cuda")
a, b = torch.cuda.Event(True), torch.cuda.Event(True)
a.record()
with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
for _ in range(40): y = x @ x
torch.cuda.current_stream().wait_stream(s1)
b.record(); torch.cuda.synchronize()
print(f"copy under GEMM load: total {a.elapsed_time(b):.1f} ms for 4 GiB copy + 40 GEMMs")
