"""Generate the committed synthetic-input fixtures under inputs/.

Calls only ``oracle/`` (the generators are Philox-driven forward simulations in
smc_oracle.cpp, tag 2).  Run once:  python -m oracle.gen_inputs
Outputs are inputs, not expected values; each file records the recipe.
"""
from __future__ import annotations

import json
import os

import numpy as np

import oracle

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "inputs")


def newick(tree):
    par, lef, rig, age = tree["parent"], tree["left"], tree["right"], tree["age"]
    names = tree.get("names")

    def rec(v):
        if lef[v] < 0:
            s = names[v] if names else f"n{v}"
        else:
            s = "(" + rec(lef[v]) + "," + rec(rig[v]) + ")"
        if par[v] >= 0:
            s += ":" + repr(round(age[par[v]] - age[v], 12))
        return s

    return rec(tree["root"]) + ";"


def tree_summary(tree):
    par, lef, rig, age = tree["parent"], tree["left"], tree["right"], tree["age"]
    M = len(age)
    total = sum(age[par[i]] - age[i] for i in range(M) if par[i] >= 0)

    def ntips(v):
        return 1 if lef[v] < 0 else ntips(lef[v]) + ntips(rig[v])

    def height(v):
        return 0 if lef[v] < 0 else 1 + max(height(lef[v]), height(rig[v]))

    def maxpend(v, pend, smaller):
        if lef[v] < 0:
            return pend
        a, b = lef[v], rig[v]
        if smaller and ntips(b) < ntips(a):
            a, b = b, a
        return max(pend + 1, maxpend(a, pend + 1, smaller), maxpend(b, pend, smaller))

    internal = sorted(age[i] for i in range(M) if lef[i] >= 0 and i != tree["root"])
    return dict(nodes=M, tips=sum(1 for i in range(M) if lef[i] < 0),
                total_branch_length=total, height_edges=height(tree["root"]),
                max_pending_left_first=maxpend(tree["root"], 0, False),
                max_pending_smaller_first=maxpend(tree["root"], 0, True),
                largest_nonroot_internal_ages=internal[-3:][::-1],
                smallest_internal_age=internal[0])


def tree5():
    # ((A:6,(B:2,C:2):4):4,(D:3,E:3):7); root age 10.
    # nodes: 0 root(10) 1 X(6) 2 A 3 W(2) 4 B 5 C 6 Y(3) 7 D 8 E
    t = dict(root=0,
             parent=[-1, 0, 1, 1, 3, 3, 0, 6, 6],
             left=[1, 2, -1, 4, -1, -1, 7, -1, -1],
             right=[6, 3, -1, 5, -1, -1, 8, -1, -1],
             age=[10.0, 6.0, 0.0, 2.0, 0.0, 0.0, 3.0, 0.0, 0.0],
             names=[None, None, "A", None, "B", "C", None, "D", "E"])
    return t


def stackf_series(D=12, seed=14):
    """Per-recursion-level observations of the STACKF program (DESIGN.md
    R-24): y_d = 1.3 + 0.3 z_d, z_d standard normal from the oracle's Philox
    uniforms (tag 2, Box-Muller with the cosine)."""
    u = oracle.uniforms(seed, 0, 0, 2, 2 * D)
    z = np.sqrt(-2.0 * np.log(u[0::2])) * np.cos(2.0 * np.pi * u[1::2])
    y = 1.3 + 0.3 * z
    with open(os.path.join(ROOT, f"stackf{D}.json"), "w") as f:
        json.dump(dict(y=y.tolist(), seed=seed,
                       recipe=f"y_d = 1.3 + 0.3 z_d, d < {D}; z_d Box-Muller of oracle.uniforms("
                              f"seed={seed}, particle 0, epoch 0, tag 2)"), f, indent=1)


def main():
    os.makedirs(ROOT, exist_ok=True)
    stackf_series()
    t5 = tree5()
    t5["newick"] = newick(t5)
    t5["summary"] = tree_summary(t5)
    t5["recipe"] = "fixed tree from SURVEY §8(c) config C0; rho = 1"
    with open(os.path.join(ROOT, "tree5.json"), "w") as f:
        json.dump(t5, f, indent=1)

    t90, used = oracle.gen_yule(90, 90, 1.0, 30.0)
    t90["names"] = [None] * len(t90["age"])
    k = 1
    for i in range(len(t90["age"])):
        if t90["left"][i] < 0:
            t90["names"][i] = f"T{k}"
            k += 1
    t90["newick"] = newick(t90)
    s = tree_summary(t90)
    s["uniforms_consumed"] = used
    t90["summary"] = s
    t90["recipe"] = ("Yule tree, oracle.gen_yule(seed=90, ntips=90, lam0=1, crown_age=30): "
                     "Philox tag 2, particle 0, epoch 0 (SURVEY §8d 'tree90')")
    with open(os.path.join(ROOT, "tree90.json"), "w") as f:
        json.dump(t90, f, indent=1)

    prm = [0.5, 1 / 4.4, 1 / 4.5, 0.5, 1 / 6.5, 0.3]
    seed = 180
    while True:
        y, z, used = oracle.gen_seir(seed, 182, prm)
        if z[:20].sum() > 0 and z[19:].sum() > 0 or z.sum() > 100:
            break
        seed += 1
    with open(os.path.join(ROOT, "seir182.json"), "w") as f:
        json.dump(dict(y=[int(v) for v in y], z_true=[int(v) for v in z], seed=seed,
                       params_true=prm, uniforms_consumed=used,
                       recipe=("oracle.gen_seir(seed, T=182, lam_h=.5, del_h=1/4.4, gam_h=1/4.5, "
                               "lam_m=.5, del_m=1/6.5, rho=.3); Philox tag 2 (SURVEY §8d 'seir182')")),
                  f, indent=1)

    for T, seed in ((10, 11), (50, 51)):
        y, x, used = oracle.gen_ssm(seed, T)
        with open(os.path.join(ROOT, f"ssm{T}.json"), "w") as f:
            json.dump(dict(y=y.tolist(), x_true=x.tolist(), seed=seed,
                           params=dict(m0=0.0, s0=100.0, drift=2.0, q=1.0, r=5.0),
                           recipe=f"oracle.gen_ssm(seed={seed}, T={T}); Eq. (2) with std devs"),
                      f, indent=1)
    print(json.dumps(s, indent=1))


if __name__ == "__main__":
    main()
