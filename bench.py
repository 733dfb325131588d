"""Benchmark: cells/s of the full QC -> normalize -> log1p -> HVG -> scale -> PCA -> kNN path.

Metric (BASELINE.json): "cells/sec end-to-end QC->kNN at 1M cells x 25k genes, 1/2/4/8 B200;
per-step ms".  One bench "step" = one pass of the whole hot path over the synthetic matrix.
Default workload = config C3 (1M cells x 25k genes, ~7.7% NB counts, H=2000, 50 PCs, k=15) on
N=1; under torchrun the same total matrix is sharded by cells over N GPUs (strong scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

``--impl reference`` times the CPU restatement (oracle/, the only CPU implementation of this
path -- the reference repo has none) on the host cores, on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cells/sec end-to-end QC→kNN at 1M cells ×25k genes, 1/2/4/8 B200; per-step ms"


def _params(args):
    from paper_2605_13928_b200.pipeline import Params
    return Params(min_genes=200, max_genes=None, max_pct_mt=20.0, min_cells=3, target_sum=1e4,
                  n_top_genes=args.hvg, n_bins=20, max_value=10.0, n_comps=50, n_neighbors=args.k,
                  regress_out=args.regress_out, connectivities=args.graph, umap=args.umap, cluster=args.cluster or args.de,
                  rank_genes=args.de)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), float(pk["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw"

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() in ("active", "1"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def _step_bytes(Z_in, N, G, Z_sub, N_sub, H, ld, regress_out=False):
    """Algorithmic HBM bytes per step."""
    return {
        "qc": 8 * Z_in + 8 * (N + 1),
        "norm_hvg": 8 * Z_in + (8 * Z_in + 8 * Z_sub) + 8 * Z_in + 4 * N,  # count, fill, hvg sums
        # scale: dense scale (its gene sums are fused into the subset fill pass of norm_hvg);
        # regress_out: dense log (8Z' + 4N ld), Aᵀl read (4N ld), in-place residual scaling (8N ld)
        "regress": (8 * Z_sub + 16 * N_sub * ld) if regress_out else (8 * Z_sub + 4 * N_sub * ld),
        "project": 4 * N_sub * ld + 4 * N_sub * 64,
    }


def cpu_baseline(args, n_sample, threads=None):
    """Time the oracle (numpy/scipy, all host cores) on the first n_sample cells of the same spec."""
    import numpy as np
    from threadpoolctl import threadpool_limits
    from oracle import pipeline as op
    from oracle.synth import SynthSpec, generate_csr, mt_mask
    cores = len(os.sched_getaffinity(0))
    spec = SynthSpec(n_sample, args.genes, seed=args.seed)
    ip, ix, d = generate_csr(spec)
    X = op.CSR(ip, ix, d, args.genes)
    p = op.Params(min_genes=200, max_genes=None, max_pct_mt=20.0, min_cells=3, n_top_genes=args.hvg,
                  n_comps=50, n_neighbors=args.k)
    with threadpool_limits(limits=threads or cores):
        t0 = time.perf_counter()
        out = op.run(X, mt_mask(spec), p, with_knn=True)
        dt = time.perf_counter() - t0
    return n_sample / dt, dt, cores, out


def bench_reference(args, rank, world):
    """--impl reference: the CPU restatement on host cores (rank 0 only under torchrun)."""
    if rank != 0:
        return
    n_sample = args.ref_sample
    vals = []
    for i in range(args.warmup + args.steps):
        v, dt, cores, _ = cpu_baseline(args, n_sample)
        if i >= args.warmup:
            vals.append((v, dt))
    value = sum(v for v, _ in vals) / len(vals)
    ms = 1e3 * sum(dt for _, dt in vals) / len(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "cells/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64/f32 (numpy)", "data": "synthetic NB counts (oracle/synth.py)",
        "config": {"workload": f"C3 sample: first {n_sample} cells x {args.genes} genes, full QC->kNN (k={args.k})",
                   "n_top_genes": args.hvg, "n_comps": 50},
        "cpu_baseline": {"value": value, "unit": "cells/s", "cores": len(os.sched_getaffinity(0)), "kind": "port",
                         "sample": f"{n_sample} cells x {args.genes} genes per step (oracle/pipeline.py run)"},
        "e2e": {"value": value, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cells", type=int, default=1_000_000)
    ap.add_argument("--genes", type=int, default=25_000)
    ap.add_argument("--hvg", type=int, default=2000)
    ap.add_argument("--k", type=int, default=15)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-sample", type=int, default=20000)
    ap.add_argument("--ref-sample", type=int, default=10000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="also build sc.pp.neighbors' distances/connectivities (umap fuzzy graph) in the step")
    ap.add_argument("--umap", action="store_true", help="also run sc.tl.umap (layout) in the step (1 GPU)")
    ap.add_argument("--cluster", action="store_true", help="also run Leiden clustering on the graph (1 GPU)")
    ap.add_argument("--de", action="store_true", help="also run Leiden + rank_genes_groups (t-test) (1 GPU)")
    ap.add_argument("--regress-out", action="store_true",
                    help="add sc.pp.regress_out(total_counts, pct_counts_mt) before scale (paper Table 1 step 4)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        bench_reference(args, rank, world)
        return

    import torch
    import torch.distributed as td
    from paper_2605_13928_b200 import _lib, pipeline, synth
    from paper_2605_13928_b200.dist import Comm, shard_rows
    from paper_2605_13928_b200.pp import DeviceCSR

    local = local % max(1, torch.cuda.device_count())  # (functional multi-rank check on one GPU)
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        # SCB_DIST_BACKEND=gloo: functional check of the multi-rank path where only one GPU is
        # available (collectives through host copies; not a timing configuration)
        backend = os.environ.get("SCB_DIST_BACKEND", "nccl")
        if backend == "nccl":
            td.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            td.init_process_group(backend)
        comm = Comm()
    p = _params(args)
    N, G = args.cells, args.genes
    r0, r1 = shard_rows(N, rank, world)
    spec = synth.Spec(N, G, seed=args.seed)

    # ---- input synthesis (untimed): this rank's rows of the global matrix
    t0 = time.time()
    X = synth.generate_rows(spec, r0, r1)
    mt = synth.mt_mask(spec)
    torch.cuda.synchronize()
    gen_s = time.time() - t0

    def barrier():
        if comm is not None:
            td.barrier()
        torch.cuda.synchronize()

    # ---- warm-up
    res = None
    for _ in range(args.warmup):
        res = None
        res = pipeline.run(X, mt, p, comm=comm, timing=False)
    barrier()

    # ---- timed region: device-resident input (14 GB >> 126 MB L2: no cache reuse across steps)
    k_start = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    k_end = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = _lib.launch_count()
    step_ms_acc = {}
    with ClockSampler(local) as clk:
        barrier()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record()
        for i in range(args.steps):
            res = None  # release the previous step's outputs before this step allocates its own
            res = pipeline.run(X, mt, p, comm=comm, timing=True, knn_timer=(k_start[i], k_end[i]))
            for kk, v in res.step_ms.items():
                step_ms_acc[kk] = step_ms_acc.get(kk, 0.0) + v
        t_end.record()
        barrier()
    launches = _lib.launch_count() - launches0
    total_ms = t_start.elapsed_time(t_end)
    if comm is not None:
        total_ms = comm.allreduce_max(total_ms)
    ms_step = total_ms / args.steps
    step_ms = {kk: v / args.steps for kk, v in step_ms_acc.items()}
    if comm is not None:
        step_ms = {kk: comm.allreduce_max(v) for kk, v in step_ms.items()}
    knn_ms = sum(a.elapsed_time(b) for a, b in zip(k_start, k_end)) / args.steps
    if comm is not None:
        knn_ms = comm.allreduce_max(knn_ms)
    value = N / (ms_step / 1e3)

    # ---- sizes for the roofline bookkeeping
    Z_in = X.nnz
    Z_total = Z_in if comm is None else comm.allreduce_int(Z_in)
    N_sub_loc = res.X_log.n_rows
    Z_sub = res.X_log.nnz
    H = int(res.hvg_index.numel())
    ld = res.scaled.ld
    n_keys = res.n_cells_total
    hbm, bf16, basis = _peaks()
    f16_peak = bf16  # dense FP16 == dense BF16 tensor rate
    flops_knn = 2.0 * N_sub_loc * n_keys * p.n_comps
    achieved = flops_knn / (knn_ms / 1e3) / 1e12
    sb = _step_bytes(Z_in, X.n_rows, G, Z_sub, N_sub_loc, H, ld, args.regress_out)
    stages = {}
    for kk in ("qc", "norm_hvg", "regress"):
        if kk in step_ms and step_ms[kk] > 0:
            stages[kk] = {"ms": round(step_ms[kk], 4), "algo_GBps": round(sb[kk] / (step_ms[kk] / 1e3) / 1e9, 1),
                          "frac_hbm": round(sb[kk] / (step_ms[kk] / 1e3) / 1e9 / hbm, 4)}
    for kk in ("pca", "knn", "graph", "umap", "cluster", "rank_genes"):
        if kk in step_ms:
            stages[kk] = {"ms": round(step_ms[kk], 4)}
    stages["knn"]["candidates_kernel_ms"] = round(knn_ms, 4)
    traffic = None  # dram bytes per launch of the kNN kernel from the committed ncu --set full capture
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01", "knn_traffic.json")
    if os.path.exists(tpath) and world == 1:
        tj = json.load(open(tpath))
        if tj.get("cells") == N and tj.get("genes") == G:
            traffic = int(tj["dram__bytes_read.sum"]) + int(tj["dram__bytes_write.sum"])
    gram_flops = float(N_sub_loc) * H * (H + 1)
    stages["pca"]["gram_flop_unique"] = gram_flops

    # ---- e2e through the public API with host buffers (H2D of the CSR + D2H of the graph)
    e2e = None
    if not args.no_e2e:
        h_indptr = torch.empty_like(X.indptr, device="cpu").pin_memory()
        h_ind = torch.empty_like(X.indices, device="cpu").pin_memory()
        h_dat = torch.empty_like(X.data, device="cpu").pin_memory()
        h_indptr.copy_(X.indptr)
        h_ind.copy_(X.indices)
        h_dat.copy_(X.data)
        # two device input buffers: the H2D copy of step i+1 (copy stream) overlaps the compute
        # of step i (compute stream); every step still copies its full input and reads back its graph
        bufs = [(torch.empty_like(X.indptr), torch.empty_like(X.indices), torch.empty_like(X.data)) for _ in range(2)]
        k = p.n_neighbors
        o_i = torch.empty((N_sub_loc, k), dtype=torch.int32).pin_memory()
        o_d = torch.empty((N_sub_loc, k), dtype=torch.float32).pin_memory()
        del X
        torch.cuda.empty_cache()
        comp = torch.cuda.current_stream()
        cs = torch.cuda.Stream()
        copied = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]

        def h2d(i):
            b = bufs[i % 2]
            with torch.cuda.stream(cs):
                if i >= 2:
                    cs.wait_event(consumed[i % 2])
                b[0].copy_(h_indptr, non_blocking=True)
                b[1].copy_(h_ind, non_blocking=True)
                b[2].copy_(h_dat, non_blocking=True)
                copied[i % 2].record(cs)

        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        h2d(0)
        for i in range(args.steps):
            if i + 1 < args.steps:
                h2d(i + 1)
            comp.wait_event(copied[i % 2])
            b = bufs[i % 2]
            Xe = DeviceCSR(b[0], b[1], b[2], G)
            r = None
            r = pipeline.run(Xe, mt, p, comm=comm, timing=False)
            consumed[i % 2].record(comp)
            if r.knn_index.shape[0] != o_i.shape[0]:
                o_i = torch.empty(tuple(r.knn_index.shape), dtype=torch.int32).pin_memory()
                o_d = torch.empty(tuple(r.knn_dist.shape), dtype=torch.float32).pin_memory()
            o_i.copy_(r.knn_index, non_blocking=True)
            o_d.copy_(r.knn_dist, non_blocking=True)
        comp.wait_stream(cs)
        e1.record(comp)
        barrier()
        e_ms = e0.elapsed_time(e1) / args.steps
        if comm is not None:
            e_ms = comm.allreduce_max(e_ms)
        h2d_bytes = h_indptr.numel() * 8 + h_ind.numel() * 4 + h_dat.numel() * 4
        d2h_bytes = o_i.numel() * 4 + o_d.numel() * 4
        e2e = {"value": N / (e_ms / 1e3), "unit": "cells/s", "ms_per_step": round(e_ms, 3),
               "h2d_bytes_per_step": int(h2d_bytes), "d2h_bytes_per_step": int(d2h_bytes),
               "overlap": "pinned H2D of step i+1 on a copy stream overlaps the compute of step i "
                          "(2 device input buffers); first copy and last compute are not overlapped"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt, cores, _ = cpu_baseline(args, args.cpu_sample)
        cpu = {"value": v, "unit": "cells/s", "cores": cores, "kind": "port",
               "sample": f"first {args.cpu_sample} cells x {G} genes of the same NB spec, full QC->kNN "
                         f"(oracle/pipeline.py, numpy/scipy BLAS on all cores), {dt:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "cells/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic NB counts generated on device (oracle/synth.py model, seed %d)" % args.seed,
            "config": {"workload": f"C3: {N} cells x {G} genes (~{Z_total / N / G:.1%} dense), full QC->normalize->"
                                   f"log1p->HVG(seurat,{args.hvg})->{'regress_out+' if args.regress_out else ''}scale->PCA(50)->"
                                   f"kNN(k={args.k}, exact){'+umap graph' if args.graph or args.umap or args.cluster or args.de else ''}{'+umap layout' if args.umap else ''}{'+leiden' if args.cluster or args.de else ''}{'+rank_genes_groups' if args.de else ''}",
                       "cells": N, "genes": G, "nnz": int(Z_total), "kept_cells": int(n_keys), "hvg": H,
                       "parallelism": f"cells sharded x{world}", "l2": "inputs (14 GB) >> L2 (126 MB); no flush needed",
                       "gen_seconds": round(gen_s, 1)},
            "step_ms": {kk: round(v, 3) for kk, v in step_ms.items()},
            "stages": stages,
            "roofline": {"kernel": "knn_candidates_kernel (tcgen05 kind::f16 distance GEMM + fused top-k)",
                         "bound": "tensor", "achieved": round(achieved, 2), "peak": round(f16_peak, 1),
                         "unit": "TFLOP/s", "frac": round(achieved / f16_peak, 4), "traffic": traffic,
                         "traffic_unit": "bytes per launch (dram read+write, ncu --set full, profiles/r01/knn_traffic.json)",
                         "algo": f"2*Nq*N*d with d={p.n_comps}: {flops_knn:.3e} FLOP per launch",
                         "peak_basis": f"{basis} dense bf16 {bf16} TFLOP/s (FP16 operands run at the BF16 rate)"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk.summary(),
            "gpu_launches": int(launches),
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        td.destroy_process_group()


if __name__ == "__main__":
    main()
