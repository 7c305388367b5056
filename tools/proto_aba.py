#!/usr/bin/env python3
"""fp64 numpy prototype of the device algorithm (design check, not shipped).

Restates one 2 ms substep the way the CUDA kernel computes it —
root-relative kinematics, segment/joint "pair" torques for J_m^T F, link
wrench for gravity + contact, and the articulated-body recursion for
M(q)^{-1}(tau - C) — and compares q̈ with the reference formulation
(oracle/msk_oracle.c: dense J_m, dense M, LDL^T).  Agreement to ~1e-10
confirms the reformulation is exact before any fp32 rounding is added.

    python tools/proto_aba.py assets/generated/wb700.json assets/generated/wb700_dance.csv
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle.oracle import OracleModel, load_clip_csv  # noqa: E402


def perp(v):
    return np.array([-v[1], v[0]])


def cross(a, b):
    return a[0] * b[1] - a[1] * b[0]


def rot(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[c, -s], [s, c]])


class Proto:
    def __init__(self, md):
        self.d = md
        self.fl = md["floating"]
        self.nrd = 3 if self.fl else 0
        self.nl = md["n_links"]
        self.nj = md["n_joints"]
        self.fc = 1 if self.fl else 0
        # parent link of every link (-1 = world/root)
        self.parent = [-1] * self.nl
        for j in range(self.nj):
            self.parent[self.fc + j] = int(md["joint_parent"][j])
        self.children = [[] for _ in range(self.nl)]
        for l in range(self.nl):
            if self.parent[l] >= 0:
                self.children[self.parent[l]].append(l)
        # pairs: (muscle, seg k, joint, endpoint k or k-1, sign)
        self.pairs = []
        for mu in range(md["n_muscles"]):
            a, b = md["m_via_start"][mu], md["m_via_start"][mu + 1]
            for v in range(a + 1, b):
                la, lb = int(md["via_link"][v - 1]), int(md["via_link"][v])
                if la == lb:
                    continue
                pa, pb = set(self.path(la)), set(self.path(lb))
                for j in sorted(pb - pa):
                    self.pairs.append((mu, v, j, v, -1.0))
                for j in sorted(pa - pb):
                    self.pairs.append((mu, v, j, v - 1, +1.0))

    def path(self, link):
        out = []
        cur = link
        while cur >= self.fc:
            j = cur - self.fc
            out.append(j)
            cur = int(self.d["joint_parent"][j])
        return out

    def qdd(self, q, dq, forces):
        d = self.d
        nl = self.nl
        # --- FK, root-relative ---
        ori = np.zeros((nl, 2))
        ang = np.zeros(nl)
        if self.fl:
            ang[0] = q[2]
        for j in range(self.nj):
            c = self.fc + j
            p = int(d["joint_parent"][j])
            po, pa = (ori[p], ang[p]) if p >= 0 else (np.zeros(2), 0.0)
            ori[c] = po + rot(pa) @ d["joint_anchor"][j]
            ang[c] = pa + d["joint_mount"][j] + q[self.nrd + j]
        O = np.array([q[0], q[1]]) if self.fl else np.zeros(2)
        # --- velocities (translation invariant) ---
        om = np.zeros(nl)
        vo = np.zeros((nl, 2))
        if self.fl:
            vo[0] = dq[0:2]
            om[0] = dq[2]
        for j in range(self.nj):
            c = self.fc + j
            p = int(d["joint_parent"][j])
            if p >= 0:
                vo[c] = vo[p] + om[p] * perp(ori[c] - ori[p])
                om[c] = om[p] + dq[self.nrd + j]
            else:
                om[c] = dq[self.nrd + j]

        def wp(l, off):
            return (np.array(off) if l < 0 else ori[l] + rot(ang[l]) @ off) if l >= 0 else np.array(off) - O

        # --- muscle pair torques ---
        tau = np.zeros(self.nrd + self.nj)
        pts = {}
        for (mu, v, j, e, sgn) in self.pairs:
            for vv in (v - 1, v):
                if vv not in pts:
                    pts[vv] = wp(int(d["via_link"][vv]), d["via_offset"][vv])
            seg = pts[v] - pts[v - 1]
            ln = np.linalg.norm(seg)
            if ln <= 1e-12:
                continue
            u = seg / ln
            r = pts[e] - ori[self.fc + j]
            tau[self.nrd + j] += sgn * forces[mu] * cross(r, u)
        # --- damping / limits ---
        for j in range(self.nj):
            k = self.nrd + j
            tau[k] -= d["joint_damping"][j] * dq[k]
            if q[k] > d["joint_hi"][j]:
                tau[k] -= d["joint_limit_stiffness"] * (q[k] - d["joint_hi"][j])
            elif q[k] < d["joint_lo"][j]:
                tau[k] -= d["joint_limit_stiffness"] * (q[k] - d["joint_lo"][j])
        # --- external wrenches at link origins: gravity + contact ---
        fext = np.zeros((nl, 3))
        g = d["gravity"]
        for l in range(nl):
            m = d["link_mass"][l]
            c = rot(ang[l]) @ np.array([d["link_com"][l], 0.0])
            F = np.array([0.0, m * g])
            fext[l] += [cross(c, F), F[0], F[1]]
        cp = d["contact"]
        for s in range(d["n_spheres"]):
            l = int(d["sphere_link"][s])
            cen = ori[l] + rot(ang[l]) @ d["sphere_offset"][s]
            pen = d["sphere_radius"][s] - (cen[1] + O[1])
            if pen <= 0:
                continue
            vc = vo[l] + om[l] * perp(cen - ori[l])
            fn = max(0.0, cp["stiffness"] * pen - cp["damping"] * vc[1])
            if fn <= 0:
                continue
            cpt = cen - np.array([0.0, d["sphere_radius"][s]])
            vcp = vo[l] + om[l] * perp(cpt - ori[l])
            ft = -cp["friction"] * fn * np.tanh(vcp[0] / cp["smoothing_vel"])
            F = np.array([ft, fn])
            fext[l] += [cross(cpt - ori[l], F), F[0], F[1]]
        # --- ABA ---
        IA = np.zeros((nl, 3, 3))
        pA = np.zeros((nl, 3))
        cb = np.zeros((nl, 3))
        for l in range(nl):
            m, I = d["link_mass"][l], d["link_inertia"][l]
            c = rot(ang[l]) @ np.array([d["link_com"][l], 0.0])
            Isp = np.array([[I + m * c @ c, -m * c[1], m * c[0]], [-m * c[1], m, 0.0], [m * c[0], 0.0, m]])
            IA[l] = Isp
            V = np.array([om[l], vo[l][0], vo[l][1]])
            h = Isp @ V
            vxf = np.array([vo[l][0] * h[2] - vo[l][1] * h[1], -om[l] * h[2], om[l] * h[1]])
            pA[l] = vxf - fext[l]
            if l >= self.fc:
                qd = dq[self.nrd + l - self.fc]
                cb[l] = [0.0, qd * vo[l][1], -qd * vo[l][0]]
        U = np.zeros((nl, 3))
        D = np.zeros(nl)
        uu = np.zeros(nl)
        for l in range(nl - 1, self.fc - 1, -1):
            j = l - self.fc
            U[l] = IA[l][:, 0]
            D[l] = IA[l][0, 0]
            uu[l] = tau[self.nrd + j] - pA[l][0]
            Ia = IA[l] - np.outer(U[l], U[l]) / D[l]
            pa = pA[l] + Ia @ cb[l] + U[l] * uu[l] / D[l]
            p = self.parent[l]
            if p < 0:
                continue
            dd = ori[l] - ori[p]
            X = np.array([[1.0, 0, 0], [-dd[1], 1.0, 0], [dd[0], 0, 1.0]])
            IA[p] += X.T @ Ia @ X
            pA[p] += X.T @ pa
        qdd = np.zeros(self.nrd + self.nj)
        A = np.zeros((nl, 3))
        if self.fl:
            A0 = np.linalg.solve(IA[0], -pA[0])
            A[0] = A0
            qdd[2] = A0[0]
            qdd[0] = A0[1] - dq[2] * dq[1]
            qdd[1] = A0[2] + dq[2] * dq[0]
        for l in range(self.fc, nl):
            p = self.parent[l]
            if p >= 0:
                dd = ori[l] - ori[p]
                Ap = A[p]
                Ai = np.array([Ap[0], Ap[1] - Ap[0] * dd[1], Ap[2] + Ap[0] * dd[0]]) + cb[l]
            else:
                Ai = cb[l].copy()
            qd = (uu[l] - U[l] @ Ai) / D[l]
            qdd[self.nrd + l - self.fc] = qd
            Ai[0] += qd
            A[l] = Ai
        return qdd, tau


def main():
    mp, cp = sys.argv[1], sys.argv[2]
    om = OracleModel(mp)
    clip = load_clip_csv(cp, om.nq, om.nk)
    pr = Proto(om.d)
    rng = np.random.default_rng(0)
    worst = 0.0
    for t in (0, 37, 500):
        q, dq = clip["q"][t].copy(), clip["dq"][t].copy()
        q[:] += rng.normal(0, 0.05, q.shape)
        dq[:] += rng.normal(0, 0.5, dq.shape)
        nm = om.nm
        act = rng.uniform(0, 1, nm)
        lm = rng.uniform(0.8, 1.2, nm)
        u = rng.uniform(0, 1, nm)
        s, qdd_ref, bad = om.substep(q, dq, act, lm, np.zeros(nm), np.zeros(nm), u)
        forces = s["f_m"]
        qdd, tau = pr.qdd(q, dq, forces)
        Jm = om.moment_arms(q)
        tau_ref = Jm.T @ forces
        e_tau = np.abs(tau[pr.nrd:] - tau_ref[pr.nrd:]).max() / max(1e-9, np.abs(tau_ref).max())
        e = np.abs(qdd - qdd_ref).max() / max(1e-9, np.abs(qdd_ref).max())
        print(f"frame {t}: rel |tau_m| err {e_tau:.3e}  rel |qdd| err {e:.3e}  (|qdd|max {np.abs(qdd_ref).max():.3g})")
        worst = max(worst, e)
    print("worst", worst)


if __name__ == "__main__":
    main()
