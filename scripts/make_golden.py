"""Write tests/golden/toy.json from the ORACLE ONLY (BASELINE.json configs[0]).

toy: sum tree 16 leaves, [T=8, B=2] buffer, n_step=3, gamma=0.99, GAE lambda=0.95,
batch 4.  Inputs are fixed literals (rewards from a small exact set, dones at
t=2 and t=T-1, S:598-style truncation); outputs are the oracle's float64 values
and ints.  Citations: S:591-599 (n-step), S:748-756 (GAE), S:346 (discounted),
S:601-629 (tree, sampling, IS weights).  Run:  python scripts/make_golden.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import philox, returns, sumtree  # noqa: E402

T, B, N_STEP, GAMMA, LAM = 8, 2, 3, 0.99, 0.95
ALPHA, BETA, EPS_P, F = 0.6, 0.4, 1e-3, 32

r = [[1.0, 0.0], [0.0, -1.0], [2.0, 0.5], [0.0, 0.0], [-1.0, 1.0], [0.5, 0.0], [0.0, 2.0], [1.0, -1.0]]
d = [[0, 0], [0, 0], [1, 0], [0, 0], [0, 1], [0, 0], [0, 0], [1, 0]]
v = [[0.5, -0.25], [1.0, 0.0], [-2.0, 1.5], [0.25, 0.75], [3.0, -1.0], [0.0, 0.5], [-0.5, 2.0], [1.25, 0.0]]
boot = [0.75, -1.5]
q_target = [[2.0, -3.0], [0.5, 1.0], [4.0, -0.5], [1.5, 10.0], [-2.0, 0.25], [3.0, 6.0], [0.0, -8.0], [7.5, 1.0]]
q_boot = [2.5, -4.0]

td = [0.5, 1.5, 0.0, 2.25, 0.125, 3.0, 0.75, 1.0, 0.25, 4.0, 0.0625, 1.25, 2.0, 0.375, 5.0, 0.875]
upd_idx = [3, 7, 3, 12]                 # a duplicate: the last write to leaf 3 wins
upd_td = [9.0, 0.0, 0.5, 6.5]
draws = philox.draws_u64(seed=2019, offset=0, n=4)


def main():
    ra, da, va = np.array(r), np.array(d, np.uint8), np.array(v)
    disc = returns.discounted_return(ra, da, np.array(boot), GAMMA)
    Rn, dn = returns.nstep_return(ra, da, N_STEP, GAMMA)
    y, _ = returns.nstep_return(ra, da, N_STEP, GAMMA, q=np.array(q_target), q_boot=np.array(q_boot))
    yr, _ = returns.nstep_return(ra, da, N_STEP, GAMMA, q=np.array(q_target), q_boot=np.array(q_boot),
                                 rescale=True, eps=1e-3)
    adv, ret = returns.gae(ra, va, da, np.array(boot), GAMMA, LAM)

    tree = sumtree.SumTreeOracle(16, F)
    tree.update(list(range(16)), td, ALPHA, EPS_P)
    q_init = list(tree.q)
    tree.update(upd_idx, upd_td, ALPHA, EPS_P)
    Q = tree.total()
    idx, qs, qmin = tree.sample(4, draws)
    w = sumtree.is_weights(qs, Q, 16, BETA)

    out = dict(
        config=dict(T=T, B=B, n_step=N_STEP, gamma=GAMMA, lam=LAM, alpha=ALPHA, beta=BETA, eps_p=EPS_P,
                    frac_bits=F, n_leaves=16, batch=4, rescale_eps=1e-3, seed=2019),
        citation="BASELINE.json configs[0]; S:346, S:591-599, S:601-629, S:748-756, S:810",
        inputs=dict(r=r, d=d, v=v, bootstrap=boot, q_target=q_target, q_boot=q_boot, td_init=td,
                    upd_idx=upd_idx, upd_td=upd_td, draws=[str(x) for x in draws]),
        discounted=disc.tolist(), nstep=Rn.tolist(), done_n=dn.tolist(), nstep_target=y.tolist(),
        nstep_target_rescaled=yr.tolist(), gae_adv=adv.tolist(), gae_ret=ret.tolist(),
        tree_q_init=[str(x) for x in q_init], tree_q=[str(x) for x in tree.q], tree_total=str(Q),
        max_seen=str(tree.max_seen), sample_idx=idx, sample_q=[str(x) for x in qs], sample_qmin=str(qmin),
        is_weights=w,
    )
    path = os.path.join(ROOT, "tests", "golden", "toy.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
