"""CPU prototype (design study, not product code): coarse spaces for the
aggregation multigrid on a C5-family Newton matrix.  Compares GMRES(50)
iteration counts of right-preconditioned GMRES with V(1,1) cycles using
(a) translation-only unsmoothed aggregation (the GPU's current coarse space)
and (b) rigid-body-mode unsmoothed aggregation (3 translations + 3 rotations
per aggregate).  argv: cells steps."""
import os, sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np, scipy.sparse as sp, scipy.sparse.linalg as spla
import bench, diffproj_oracle as O
from paper_2603_16478_b200 import core

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
sc = bench.make_scene(n, fingers=True)
osc = O.OScene(core.scene_to_arrays(sc)); els = O.build_elements(osc); A0 = O.assemble_A(osc, els)
st = sc.rest_state(); q, v = st.q.copy(), st.v.copy()
for k in range(steps):
    bench.move_fingers(sc, k)
    osc = O.OScene(core.scene_to_arrays(sc))
    o = O.forward_step(osc, A0, els, q, v, O.ForwardConfig(tol=1e-10))
    q, v = o.q_new, o.v_new
ct = O.detect_contacts(osc, q)
es = O.project_elements(els, q, True)
O.solve_multipliers(ct, q, q)
Ah = sp.csr_matrix(O.newton_matrix(osc, A0, els, es, ct))
N = Ah.shape[0] // 3
X = q.reshape(-1, 3)
print("ndof", Ah.shape[0], "nnz", Ah.nnz, "contacts", len(ct.vertex))
import os as _os

# block graph and greedy aggregation (same two-phase algorithm as dp_mg.cu)
B = sp.csr_matrix((np.ones(Ah.nnz), Ah.indices // 3, Ah.indptr[::3][:len(Ah.indptr[::3])]), shape=(N, Ah.shape[1]))
G = (abs(Ah) @ sp.kron(sp.eye(N), np.ones((3, 1))).tocsr())
G = sp.csr_matrix((sp.kron(sp.eye(N), np.ones((1, 3))) @ G) != 0)


def aggregate(G):
    n = G.shape[0]
    agg = -np.ones(n, int)
    na = 0
    for i in range(n):
        if agg[i] >= 0:
            continue
        nb = G.indices[G.indptr[i]:G.indptr[i + 1]]
        if np.any(agg[nb] >= 0):
            continue
        agg[nb] = na
        agg[i] = na
        na += 1
    tmp = agg.copy()
    for i in range(n):
        if agg[i] >= 0:
            continue
        nb = G.indices[G.indptr[i]:G.indptr[i + 1]]
        a = agg[nb]
        a = a[a >= 0]
        if len(a):
            vals, cnt = np.unique(a, return_counts=True)
            tmp[i] = vals[np.argmax(cnt)]
    agg = tmp
    for i in range(n):
        if agg[i] < 0:
            agg[i] = na
            nb = G.indices[G.indptr[i]:G.indptr[i + 1]]
            for j in nb:
                if agg[j] < 0:
                    agg[j] = na
            na += 1
    return agg, na


def skew(r):
    return np.array([[0, -r[2], r[1]], [r[2], 0, -r[0]], [-r[1], r[0], 0]])


def prolong(agg, na, X, rbm):
    rows, cols, vals = [], [], []
    bs = 6 if rbm else 3
    cent = np.zeros((na, 3)); cnt = np.zeros(na)
    np.add.at(cent, agg, X); np.add.at(cnt, agg, 1); cent /= cnt[:, None]
    for i in range(len(agg)):
        I = agg[i]
        blk = np.eye(3) if not rbm else np.hstack([np.eye(3), -skew(X[i] - cent[I])])
        for a in range(3):
            for b in range(bs):
                rows.append(3 * i + a); cols.append(bs * I + b); vals.append(blk[a, b])
    return sp.csr_matrix((vals, (rows, cols)), shape=(3 * len(agg), bs * na)), cent


def block_jacobi_inv(A, bs):
    n = A.shape[0] // bs
    D = np.zeros((n, bs, bs))
    Ad = A.tocsr()
    for i in range(n):
        D[i] = Ad[bs * i:bs * i + bs, bs * i:bs * i + bs].toarray()
    Dinv = np.linalg.inv(D)
    return sp.block_diag(list(Dinv), format='csr')


def build(Ah, X, rbm, levels):
    lv = []
    A = Ah; Xc = X; bs = 3
    G0 = G
    for l in range(levels - 1):
        agg, na = aggregate(G0 if l == 0 else Gc)
        if l == 0:
            P, cent = prolong(agg, na, Xc, rbm)
        else:
            # coarse-to-coarser: translations/rotations of aggregates of aggregates
            cbs = 6 if rbm else 3
            rows, cols, vals = [], [], []
            cent2 = np.zeros((na, 3)); cnt = np.zeros(na)
            np.add.at(cent2, agg, Xc); np.add.at(cnt, agg, 1); cent2 /= cnt[:, None]
            for i in range(len(agg)):
                I = agg[i]
                if rbm:
                    blk = np.eye(6); blk[:3, 3:] = -skew(Xc[i] - cent2[I])
                else:
                    blk = np.eye(3)
                for a in range(cbs):
                    for b in range(cbs):
                        if blk[a, b] != 0:
                            rows.append(cbs * i + a); cols.append(cbs * I + b); vals.append(blk[a, b])
            P = sp.csr_matrix((vals, (rows, cols)), shape=(cbs * len(agg), cbs * na))
            cent = cent2
        Dinv = block_jacobi_inv(A, bs)
        if SMOOTH_P:
            # smoothed aggregation: P = (I - w D^-1 A) P0, w = 4/(3 rho(D^-1 A))
            DA = Dinv @ A
            rho = abs(spla.eigs(DA, k=1, which='LM', return_eigenvectors=False, maxiter=200, tol=1e-2)[0])
            P = (P - (4.0 / (3.0 * rho)) * (DA @ P)).tocsr()
        Ac = (P.T @ A @ P).tocsr()
        lv.append((A, Dinv, P))
        bs = 6 if rbm else 3
        # coarse block graph
        Gc = sp.csr_matrix((sp.kron(sp.eye(na), np.ones((1, bs))) @ (abs(Ac) @ sp.kron(sp.eye(na), np.ones((bs, 1))))) != 0)
        A = Ac; Xc = cent
    lv.append((A, None, None))
    return lv


SMOOTHER = os.environ.get("SMOOTHER", "jacobi")
_colors = {}


def colors_for(A, bs):
    key = id(A)
    if key not in _colors:
        n = A.shape[0] // bs
        Gb = sp.csr_matrix((sp.kron(sp.eye(n), np.ones((1, bs))) @ (abs(A) @ sp.kron(sp.eye(n), np.ones((bs, 1))))) != 0)
        col = -np.ones(n, int)
        for i in range(n):
            nb = Gb.indices[Gb.indptr[i]:Gb.indptr[i + 1]]
            used = set(col[nb][col[nb] >= 0].tolist())
            c = 0
            while c in used:
                c += 1
            col[i] = c
        _colors[key] = [np.concatenate([np.arange(bs * i, bs * i + bs) for i in np.nonzero(col == c)[0]])
                        for c in range(col.max() + 1)]
    return _colors[key]


def smooth_step(A, Dinv, b, x, omega, bs, level=0):
    if SMOOTHER == "jacobi" or (SMOOTHER == "mcgs0" and level > 0):
        return x + omega * (Dinv @ (b - A @ x))
    # multicolour block Gauss-Seidel, one forward sweep
    x = x.copy()
    for idx in colors_for(A, bs):
        r = b[idx] - A[idx] @ x
        x[idx] += (Dinv[idx][:, idx] @ r)
    return x


def vcycle(lv, l, b, omega=0.8, alpha=1.5):
    A, Dinv, P = lv[l]
    if P is None:
        return spla.spsolve(A.tocsc(), b)
    bs = 3 if l == 0 else (Dinv.shape[0] // (A.shape[0] // 3) * 3 if False else 3)
    x = smooth_step(A, Dinv, b, np.zeros_like(b), omega, bs, l)
    r = b - A @ x
    xc = vcycle(lv, l + 1, P.T @ r, omega, alpha)
    x = x + alpha * (P @ xc)
    if os.environ.get("POST0") and l == 0:
        return x
    x = smooth_step(A, Dinv, b, x, omega, bs, l)
    return x


def gmres_count(Ah, M, tol, restart=50):
    b = np.random.default_rng(0).standard_normal(Ah.shape[0])
    it = [0]
    def cb(_):
        it[0] += 1
    Mop = spla.LinearOperator(Ah.shape, matvec=M)
    # right preconditioning via A M y = b
    AM = spla.LinearOperator(Ah.shape, matvec=lambda y: Ah @ M(y))
    y, info = spla.gmres(AM, b, rtol=tol, restart=restart, maxiter=2000, callback=cb, callback_type='pr_norm')
    return it[0], info


import os
SMOOTH_P = os.environ.get("SA") == "1"
for rbm in (False,):
    for alpha in ((1.0,) if SMOOTH_P else (1.0, 1.5)):
        for levels in (3,):
            t0 = time.time()
            lv = build(Ah, X, rbm, levels)
            M = lambda r, lv=lv, alpha=alpha: vcycle(lv, 0, r, 0.8, alpha)
            res = [gmres_count(Ah, M, tol) for tol in (1e-3, 1e-10)]
            print(f"smoother={SMOOTHER} SA={SMOOTH_P} nnz(Ac)={lv[1][0].nnz} rbm={rbm} alpha={alpha} levels={levels} coarse={lv[1][0].shape[0]} iters(1e-3,1e-10)={[r[0] for r in res]} t={time.time()-t0:.1f}s", flush=True)
