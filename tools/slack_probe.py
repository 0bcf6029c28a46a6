import os, sys, json
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2107_09801_b200 as P
from conftest import load_golden
for L in ("16383", "65535"):
    g = load_golden("kats.json")[L]
    for slack in ("1e-6", "1e-5", "3e-5", "1e-4", "3e-4", "1e-3"):
        os.environ["PSLB200_CERT_SLACK"] = slack
        ctx = P.default_context(); b = ctx.scan_stats()
        p = P.SearchParams(length=g["params"][0], seed=g["params"][1], alpha1=4, alpha2=g["params"][3], ls_lmt=g["params"][4], flip_lmt=10, n_lmt=1024, stop=P.StopCondition(max_nse=g["params"][7]))
        r = P.run_search(p)
        a = ctx.scan_stats()
        print(L, slack, {k: a[k]-b[k] for k in a}, r.nse == g["nse"] and r.psl_best == g["psl_best"])
