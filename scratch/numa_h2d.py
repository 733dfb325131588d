# Pinned H2D bandwidth vs the NUMA node the pinned pages live on (first touch by a thread bound
# to that node's CPUs).  Prints the GPU's NUMA node, each node's CPU list and GB/s.
import os, glob, time, torch
props = torch.cuda.get_device_properties(0)
bus = "%04x:%02x:%02x.0" % (props.pci_domain_id, props.pci_bus_id, props.pci_device_id)
try:
    gpu_node = int(open(f"/sys/bus/pci/devices/{bus}/numa_node").read())
except Exception as e:
    gpu_node = f"? ({e})"
print("gpu", bus, "numa_node", gpu_node)
def cpulist(s):
    out = []
    for part in s.strip().split(","):
        if "-" in part:
            a, b = part.split("-"); out += list(range(int(a), int(b) + 1))
        elif part:
            out.append(int(part))
    return out
nodes = {}
for d in sorted(glob.glob("/sys/devices/system/node/node[0-9]*")):
    nodes[int(d.rsplit("node", 1)[1])] = cpulist(open(d + "/cpulist").read())
allowed = os.sched_getaffinity(0)
print("nodes", {k: (len(v), len(set(v) & allowed)) for k, v in nodes.items()}, "allowed", len(allowed))
n = 1 << 30  # 4 GiB float32
d = torch.empty(n, dtype=torch.float32, device="cuda")
for node, cpus in nodes.items():
    cs = set(cpus) & allowed
    if not cs:
        continue
    os.sched_setaffinity(0, cs)
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    h.fill_(1.0)
    best = 0
    for rep in range(3):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); d.copy_(h, non_blocking=True); b.record(); torch.cuda.synchronize()
        best = max(best, 4 * n / a.elapsed_time(b) / 1e6)
    print(f"pinned pages first-touched on node {node}: H2D {best:.1f} GB/s", flush=True)
    del h
os.sched_setaffinity(0, allowed)
