import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import paper_2501_07642_b200 as frr, oracle as O
which = sys.argv[1]
if which == "regen":
    for n, t in [(2, 1), (10, 7), (1000, 500)]:
        d = np.arange(50, dtype=np.uint64)
        ok = np.array_equal(frr.batch_assignments(3, d, n, t), O.c_batch_assign(3, d, n, t))
        print("regen", n, t, ok, flush=True)
elif which == "nt":
    os.environ["FRR_MC_PATH"] = "tensor_core"
    for n, d, t, M in [(300, 200, 150, 3000), (2000, 1024, 1000, 2048), (1000, 1001, 17, 1000)]:
        X = np.random.default_rng(2).standard_normal((n, d))
        design = frr.DesignSpec(n, t, accept_prob=1.0, max_draws=M, batch_size=M, root_seed=42, precision_mode="ridge")
        kern = frr.precompute_precision(X, "ridge")._kernel
        st = frr.generation.mc_stats_device(kern, design, 0, M).cpu().numpy()
        want = O.c_mc_stats(O.Balance(kern._zq, kern._inv_scale_sq), t, 42, 0, M)
        print("nt", n, d, int((st.view(np.uint64) != want.view(np.uint64)).sum()), "mismatches", flush=True)
