import torch
a = torch.load("/tmp/knn_tau0.pt"); b = torch.load("/tmp/knn_tau1.pt")
same = (a["idx"] == b["idx"]).all(dim=1)
print(f"[cmp] rows identical {same.float().mean().item():.6f}, max |dd| {(a['d']-b['d']).abs().max().item():.3g}")
sa = torch.sort(a["idx"], 1).values; sb = torch.sort(b["idx"], 1).values
print(f"[cmp] neighbour sets identical {(sa == sb).all(1).float().mean().item():.6f}")
