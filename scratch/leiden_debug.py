import sys; sys.path.insert(0, ".")
import numpy as np, torch
from tests.test_gpu_cluster import _graph
from paper_2605_13928_b200 import pp
G, truth = _graph(n=1500, k=6, seed=11)
print(pp.leiden(G, seed=3)[1:])
