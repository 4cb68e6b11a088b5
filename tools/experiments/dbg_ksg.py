import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from tests.gpu_utils import Case
from paper_2208_09822_b200 import iaat
def force(**kw):
    for k in list(os.environ):
        if k.startswith("IAAT_FORCE_"): os.environ.pop(k)
    for k, v in kw.items(): os.environ["IAAT_FORCE_" + k.upper()] = str(v)
ents = [e for e in iaat.iaat_catalog_describe() if e["family"] == "ksg" and e["trans"] == "NN"]
for e in ents:
  for (M,N,K,beta) in [(61,70,50,0.5),(61,70,50,0.0),(44,52,37,0.5),(80,36,100,0.5),(61,70,48,0.5),(61,64,48,0.5),(64,70,48,0.5)]:
    force(family=7, order=e["index"])
    c = Case(np.float32, "N", "N", M, N, K, 301, 31, 1.5, beta, ld_multiple=4)
    p = iaat.iaat_plan_describe(0, "N", "N", M, N, K, c.lda, c.sA, c.ldb, c.sB, c.ldc, c.sC, c.batch, beta == 0)
    if p.get("family") != "ksg" or p.get("entry") != e["index"]: continue
    c.run(); torch.cuda.synchronize()
    got = c.views()[2].clone()
    force(family=0)
    c2 = Case(np.float32, "N", "N", M, N, K, 301, 31, 1.5, beta, ld_multiple=4)
    c2.run(); torch.cuda.synchronize()
    ref = c2.views()[2]
    a, b = got.view(torch.int32), ref.view(torch.int32)
    bad = (a != b).nonzero().flatten()
    msg = "OK"
    if len(bad):
        i = bad[:5].tolist()
        locs = [(x // c.sC, (x % c.sC) % c.ldc, (x % c.sC) // c.ldc) for x in i]
        msg = "BAD %d: %s got %s ref %s" % (len(bad), locs, got[bad[:5]].tolist(), ref[bad[:5]].tolist())
    print(e["mr"], e["nr"], e["lr"], e["kc"], e["g"], e["w"], (M, N, K, beta), "Mv", p["Mv"], "Nv", p["Nv"], "P", p["P"], msg, flush=True)
force()
