import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import paper_2210_03523_b200 as dg
import oracle as orc
orc.build()
from test_gpu_curved import setup
from test_gpu_parity import tau_rel
kernels = ("grp", "ext", "generic")
names = sys.argv[1:] or ["cfg4_small", "cfg5_subbox", "cfg4_full"]
for name, kern in [(n, k) for n in names for k in kernels]:
    os.environ.pop("DGTAU_TAU_GENERIC", None)
    os.environ.pop("DGTAU_TAU_PERLEVEL", None)
    if kern == "generic":
        os.environ["DGTAU_TAU_GENERIC"] = "1"
    if kern == "ext":
        os.environ["DGTAU_TAU_PERLEVEL"] = "1"
    for ref in ("solver", "same"):
        for form in (0, 1):
            mesh, orders, P, S, q, qd = setup(dg, orc, name)
            if ref == "solver":
                tg = S.tau_estimate(qd, S.rhs_eval(qd), formulation=form, reference=dg.REF_SOLVER).cpu().numpy()
                to = P.tau_estimate(orders, q, P.rhs(orders, q), form)
            else:
                tg = S.tau_estimate(qd, None, formulation=form, reference=dg.REF_SAME).cpu().numpy()
                to = P.tau_estimate(orders, q, P.rhs(orders, q, orc.ISOLATED), form)
            print(name, kern, ref, form, "%.2e" % tau_rel(tg, to))
