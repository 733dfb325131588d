# eigensolve timing on the real pipeline's scaled matrix (synthetic NB counts), several filter degrees
import os, sys, torch, subprocess
sys.path.insert(0, ".")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300000
if len(sys.argv) > 2:
    from paper_2605_13928_b200 import synth, pipeline, pp
    spec = synth.Spec(n, 25000, seed=0)
    X = synth.generate(spec); mt = synth.mt_mask(spec)
    r = pipeline.run(X, mt, pipeline.Params(), with_knn=False)
    sc = r.scaled
    C = pp.gram(sc)
    N = sc.Z.shape[0]
    for i in range(3):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); lam, comp_t, mean, tr = pp.pca_from_gram(sc, C, N, 50); b.record(); torch.cuda.synchronize()
        print("deg", os.environ.get("SCB_EIG_DEGREE"), "eig total", round(a.elapsed_time(b), 2), "ms lam", lam[:2].tolist(), lam[48:50].tolist(), flush=True)
        if i == 0:
            torch.save(comp_t.cpu(), f"/tmp/comp_{os.environ.get('SCB_EIG_DEGREE')}.pt")
else:
    for deg in (3, 5, 6, 8):
        env = dict(os.environ, SCB_EIG_DEGREE=str(deg), SCB_EIG_VERBOSE="1")
        subprocess.run([sys.executable, __file__, str(n), "run"], env=env)
    import torch
    ref = torch.load("/tmp/comp_3.pt").double()
    for deg in (5, 6, 8):
        c = torch.load(f"/tmp/comp_{deg}.pt").double()
        print(deg, "max |cos| deviation", (1 - (ref[:50] * c[:50]).sum(1).abs()).max().item())
