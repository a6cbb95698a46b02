import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import synth, oracle
import paper_1802_10291_b200 as m
c = synth.CONFIGS[3]
g = synth.cfg3_rows(np.arange(4)).copy()
g[1] = np.random.default_rng(11).standard_normal(g[1].shape).astype(np.float32) * 3.0
P = oracle.OraclePlan(c["M"], c["N"], c["L"], c["bank"])
ref_f = P.eval(g[[1]]); ref_h = P.eval(g[[1]], hilbert=True)
def rel(a, b): return np.linalg.norm(a - b) / np.linalg.norm(b)
for env in [{}, {"MCI_ROW_QTAB": "1"}, {"MCI_DISABLE_ROW": "1"}]:
    for k in ("MCI_ROW_QTAB", "MCI_DISABLE_ROW"): os.environ.pop(k, None)
    os.environ.update(env)
    plan = m.Plan(c["M"], c["N"], c["L"], c["bank"], hilbert=True)
    gd = torch.from_numpy(g).cuda()
    f, hf = plan.execute(gd); torch.cuda.synchronize()
    f = f.double().cpu().numpy(); hf = hf.double().cpu().numpy()
    print(env, plan.path, "f rel", rel(f[1], ref_f[0]), "hf rel", rel(hf[1], ref_h[0]), "|f|", np.linalg.norm(ref_f[0]) / 256)
