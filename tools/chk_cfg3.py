import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, oracle, workloads as W, paper_2210_03523_b200 as dg
oracle.build()
mesh = W.cube_mesh(32); orders = W.orders_random(mesh.E, 2, 7, 3)
P = oracle.Problem(mesh); X = P.node_coords(orders); q = W.pulse_state(X, orders, sigma=0.1)
S = dg.Solver(mesh); S.set_orders(orders)
r = S.rhs_eval(torch.from_numpy(q).cuda()).cpu().numpy(); ro = P.rhs(orders, q)
off = W.offsets(orders)
for v in range(5):
    g=[];o=[]
    for e in range(len(orders)):
        n=(off[e+1]-off[e])//5
        g.append(r[off[e]:off[e+1]].reshape(5,n)[v]); o.append(ro[off[e]:off[e+1]].reshape(5,n)[v])
    g=np.concatenate(g); o=np.concatenate(o)
    print(v, "max|orc|", np.abs(o).max(), "max|diff|", np.abs(g-o).max(), "rel", np.abs(g-o).max()/np.abs(o).max())
# locate the largest energy-residual differences
errs=[]
for e in range(len(orders)):
    n=(off[e+1]-off[e])//5
    d=np.abs(r[off[e]:off[e+1]].reshape(5,n)-ro[off[e]:off[e+1]].reshape(5,n))
    errs.append((d.max(), e, int(np.unravel_index(d.argmax(), d.shape)[0]), int(np.unravel_index(d.argmax(), d.shape)[1])))
errs.sort(reverse=True)
for m,e,v,node in errs[:8]:
    N=orders[e]; n1,n2=N[0]+1,N[1]+1
    i=node%n1; j=(node//n1)%n2; k=node//(n1*n2)
    print(f"e={e} N={tuple(N)} var={v} node=({i},{j},{k}) err={m:.3e} nbr_orders=", [tuple(orders[x]) for x in mesh.nbr[e]])
# isolated variant (no faces)
ri = S.rhs_eval(torch.from_numpy(q).cuda(), variant=1).cpu().numpy(); roi = P.rhs(orders, q, oracle.ISOLATED)
print("isolated max diff", np.abs(ri-roi).max())
