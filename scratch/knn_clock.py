# sample SM clock / power while the kNN candidate kernel runs back to back
import sys, time, threading, subprocess, torch
sys.path.insert(0, ".")
from paper_2605_13928_b200 import pp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
g = torch.Generator(device="cuda"); g.manual_seed(0)
sig = torch.linspace(4.0, 0.6, 50, device="cuda")
centers = torch.randn(30, 50, device="cuda", generator=g) * sig * 1.5
lab = torch.randint(0, 30, (n,), device="cuda", generator=g)
X = (centers[lab] + torch.randn(n, 50, device="cuda", generator=g) * sig * 0.6).contiguous()
pp.neighbors(X, 15); torch.cuda.synchronize()
out = []
stop = threading.Event()
def sampler():
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active", "--format=csv,noheader"],
                           capture_output=True, text=True).stdout.strip()
        out.append(r); time.sleep(0.05)
th = threading.Thread(target=sampler); th.start()
t = (torch.cuda.Event(True), torch.cuda.Event(True))
t0 = time.time()
for i in range(12):
    pp.neighbors(X, 15, timer=t)
torch.cuda.synchronize()
stop.set(); th.join()
print(f"12 knn in {time.time()-t0:.2f}s, last candidates {t[0].elapsed_time(t[1]):.1f} ms")
for o in out: print(o)
