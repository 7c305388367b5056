#!/usr/bin/env python3
"""Deterministic generators for the models and clips the reference does not ship.

The reference bundles no model or clip files (its ``examples/`` and
``vendor/`` are git-ignored, /root/reference/proj/.gitignore:1-2), so every
workload in BASELINE.json is authored here in the reference's own schemas:

* model JSON  — keys accepted by ``parse_model_json`` (/root/reference/proj/src/model.cpp:94-196)
  and valid under ``ModelSpec::validate`` (model.cpp:18-86);
* clip CSV    — the column layout of ``load_reference`` / ``save_reference``
  (/root/reference/proj/src/reference.cpp:35-130), 50 Hz, ``%.17g``.

Key-body columns are produced by forward kinematics identical to
``forward_kinematics`` + ``key_body_state`` (skeleton.cpp:82-107, 346-357) so
that the tracking error is zero on every clip frame.

Models: pendulum1_m2, arm2_m6, walker5_m16, and the
whole-body planar humanoid wb700 (floating root, 80 links, 700 muscles,
10 key bodies, 10 contact spheres) with its pinned-pelvis twin wb700_fixed
(SURVEY.md Appendix B).  Clips: a filtered sinusoid for the small models,
``dance`` and ``backflip`` for the whole-body model.

Usage:  python tools/gen_assets.py [--out assets/generated]
"""
from __future__ import annotations

import argparse
import json
import math
import os
from dataclasses import dataclass, field

import numpy as np

RATE = 50.0
CTRL_DT = 0.02


# --------------------------------------------------------------------------
# model description helpers
# --------------------------------------------------------------------------
@dataclass
class Link:
    name: str
    length: float
    mass: float
    inertia: float
    com: float


@dataclass
class Joint:
    name: str
    child: int
    parent: int
    anchor: tuple
    mount_angle: float = 0.0
    limits: tuple = (-3.0, 3.0)
    damping: float = 0.0


@dataclass
class Model:
    name: str
    root: str
    links: list = field(default_factory=list)
    joints: list = field(default_factory=list)
    muscles: list = field(default_factory=list)
    spheres: list = field(default_factory=list)
    key_bodies: list = field(default_factory=list)
    contact: dict | None = None
    gravity: float = -9.81
    joint_limit_stiffness: float = 200.0

    @property
    def floating(self):
        return self.root == "floating"

    @property
    def nrd(self):
        return 3 if self.floating else 0

    @property
    def nq(self):
        return self.nrd + len(self.joints)

    def to_json(self):
        d = {
            "name": self.name,
            "root": self.root,
            "gravity": self.gravity,
            "joint_limit_stiffness": self.joint_limit_stiffness,
            "links": [
                {"name": l.name, "length": l.length, "mass": l.mass, "inertia": l.inertia, "com": l.com}
                for l in self.links
            ],
            "joints": [
                {
                    "name": j.name,
                    "child": j.child,
                    "parent": j.parent,
                    "anchor": [j.anchor[0], j.anchor[1]],
                    "mount_angle": j.mount_angle,
                    "limits": [j.limits[0], j.limits[1]],
                    "damping": j.damping,
                }
                for j in self.joints
            ],
            "muscles": self.muscles,
            "key_bodies": self.key_bodies,
        }
        if self.contact is not None or self.spheres:
            c = dict(self.contact or {})
            c["spheres"] = self.spheres
            d["contacts"] = c
        return d


# --------------------------------------------------------------------------
# kinematics (restates skeleton.cpp:82-113 and 346-357 for data generation)
# --------------------------------------------------------------------------
def rot(a):
    c, s = math.cos(a), math.sin(a)
    return np.array([[c, -s], [s, c]])


def fk(model: Model, q):
    nl = len(model.links)
    origin = [np.zeros(2) for _ in range(nl)]
    angle = [0.0] * nl
    anchors = [np.zeros(2) for _ in model.joints]
    fc = 1 if model.floating else 0
    if model.floating:
        origin[0] = np.array([q[0], q[1]])
        angle[0] = q[2]
    for j, jt in enumerate(model.joints):
        c = fc + j
        po, pa = (origin[jt.parent], angle[jt.parent]) if jt.parent >= 0 else (np.zeros(2), 0.0)
        aw = po + rot(pa) @ np.array(jt.anchor)
        anchors[j] = aw
        origin[c] = aw
        angle[c] = pa + jt.mount_angle + q[model.nrd + j]
    return origin, angle, anchors


def world_point(origin, angle, link, local):
    if link < 0:
        return np.array(local, dtype=float)
    return origin[link] + rot(angle[link]) @ np.array(local, dtype=float)


def ground_offset(model: Model, q):
    """Clip-pipeline ground correction (SPEC.md clip pipeline: minimum foot
    height across the entire sequence): shift the root height so the lowest
    contact-sphere bottom over the whole clip touches z = 0."""
    if not model.floating or not model.spheres:
        return q
    low = np.inf
    for row in q:
        origin, angle, _ = fk(model, row)
        for sp in model.spheres:
            p = world_point(origin, angle, sp["link"], sp["offset"])
            low = min(low, p[1] - sp["radius"])
    q = q.copy()
    q[:, 1] -= low
    return q


def key_body_state(model, origin, angle):
    pos, ang = [], []
    for l in model.key_bodies:
        pos.append(world_point(origin, angle, l, (model.links[l].com, 0.0)))
        ang.append(angle[l])
    return pos, ang


def mtu_len(model, origin, angle, vps):
    pts = [world_point(origin, angle, v[0], v[1]) for v in vps]
    return float(sum(np.linalg.norm(pts[k] - pts[k - 1]) for k in range(1, len(pts))))


def subtree(model: Model, link: int):
    fc = 1 if model.floating else 0
    out = [link]
    for j, jt in enumerate(model.joints):
        c = fc + j
        if jt.parent in out and c not in out:
            out.append(c)
    return out


def joint_local_inertia(model: Model, joint: int, q0):
    """Smaller of the parent's and child's rotational inertia about the joint."""
    origin, angle, anchors = fk(model, q0)
    fc = 1 if model.floating else 0
    a = anchors[joint]
    vals = []
    for l in (model.joints[joint].parent, fc + joint):
        if l < 0:
            continue
        lk = model.links[l]
        c = world_point(origin, angle, l, (lk.com, 0.0))
        vals.append(lk.inertia + lk.mass * float(np.sum((c - a) ** 2)))
    return min(vals)


def moment_arms_fd(model: Model, vps, q0, joints, h=1e-6):
    """|dL/dq_j| by central differences at q0 (used only to size f_max)."""
    out = []
    for j in joints:
        d = model.nrd + j
        qp, qm = np.array(q0, dtype=float), np.array(q0, dtype=float)
        qp[d] += h
        qm[d] -= h
        op, ap, _ = fk(model, qp)
        om, am, _ = fk(model, qm)
        out.append(abs(mtu_len(model, op, ap, vps) - mtu_len(model, om, am, vps)) / (2 * h))
    return out


def joint_eff_inertia(model: Model, joint: int, q0):
    """Composite rotational inertia of the child subtree about the joint."""
    origin, angle, anchors = fk(model, q0)
    fc = 1 if model.floating else 0
    a = anchors[joint]
    tot = 0.0
    for l in subtree(model, fc + joint):
        lk = model.links[l]
        c = world_point(origin, angle, l, (lk.com, 0.0))
        tot += lk.inertia + lk.mass * float(np.sum((c - a) ** 2))
    return tot


# --------------------------------------------------------------------------
# muscle helper
# --------------------------------------------------------------------------
def make_muscle(model, name, vps, q0, f_max, v_max=10.0, tau_act=0.010, tau_deact=0.040, lopt_frac=0.6):
    origin, angle, _ = fk(model, q0)
    L = mtu_len(model, origin, angle, vps)
    l_opt = lopt_frac * L
    slack = L - l_opt  # normalised fibre length 1 at the neutral pose
    return {
        "name": name,
        "f_max": float(f_max),
        "l_opt": float(l_opt),
        "v_max": float(v_max),
        "tau_act": float(tau_act),
        "tau_deact": float(tau_deact),
        "tendon_slack": float(slack),
        "via_points": [[int(v[0]), [float(v[1][0]), float(v[1][1])]] for v in vps],
    }


# --------------------------------------------------------------------------
# small models
# --------------------------------------------------------------------------
def pendulum1_m2():
    m = Model("pendulum1_m2", "fixed")
    m.links = [Link("link", 0.5, 1.0, 1.0 * 0.5**2 / 12, 0.25)]
    m.joints = [Joint("hinge", 0, -1, (0.0, 0.0), -math.pi / 2, (-2.5, 2.5), 0.02)]
    q0 = np.zeros(1)
    m.muscles = [
        make_muscle(m, "flexor", [(-1, (0.06, 0.04)), (0, (0.2, 0.03))], q0, 120.0),
        make_muscle(m, "extensor", [(-1, (-0.06, 0.04)), (0, (0.2, -0.03))], q0, 120.0),
    ]
    m.key_bodies = [0]
    return m


def arm2_m6():
    m = Model("arm2_m6", "fixed")
    m.links = [
        Link("upper_arm", 0.30, 2.0, 2.0 * 0.30**2 / 12, 0.15),
        Link("forearm", 0.28, 1.4, 1.4 * 0.28**2 / 12, 0.13),
    ]
    m.joints = [
        Joint("shoulder", 0, -1, (0.0, 0.0), -math.pi / 2, (-2.0, 2.0), 0.05),
        Joint("elbow", 1, 0, (0.30, 0.0), 0.0, (-0.05, 2.6), 0.03),
    ]
    q0 = np.array([0.3, 0.9])
    m.muscles = [
        make_muscle(m, "shoulder_flexor", [(-1, (0.05, 0.03)), (0, (0.12, 0.025))], q0, 600.0),
        make_muscle(m, "shoulder_extensor", [(-1, (-0.05, 0.03)), (0, (0.12, -0.025))], q0, 600.0),
        make_muscle(m, "elbow_flexor", [(0, (0.10, 0.02)), (1, (0.05, 0.015))], q0, 450.0),
        make_muscle(m, "elbow_extensor", [(0, (0.12, -0.02)), (1, (-0.02, -0.012))], q0, 450.0),
        make_muscle(m, "biarticular_flexor", [(-1, (0.03, 0.02)), (0, (0.15, 0.03)), (1, (0.06, 0.015))], q0, 300.0),
        make_muscle(m, "biarticular_extensor", [(-1, (-0.03, 0.02)), (0, (0.15, -0.03)), (1, (-0.02, -0.012))], q0, 300.0),
    ]
    m.key_bodies = [0, 1]
    return m


def walker5_m16():
    m = Model("walker5_m16", "floating")
    m.joint_limit_stiffness = 200.0
    m.contact = {"stiffness": 2.0e4, "damping": 300.0, "friction": 0.9, "smoothing_vel": 0.05}
    m.links = [
        Link("torso", 0.60, 30.0, 30.0 * 0.6**2 / 12, 0.30),
        Link("thigh_l", 0.45, 7.0, 7.0 * 0.45**2 / 12, 0.20),
        Link("shank_l", 0.45, 3.5, 3.5 * 0.45**2 / 12, 0.20),
        Link("thigh_r", 0.45, 7.0, 7.0 * 0.45**2 / 12, 0.20),
        Link("shank_r", 0.45, 3.5, 3.5 * 0.45**2 / 12, 0.20),
    ]
    # torso local x points up when q2 = pi/2; hips at the proximal end.
    m.joints = [
        Joint("hip_l", 1, 0, (0.0, 0.0), math.pi, (-2.2, 1.2), 0.5),
        Joint("knee_l", 2, 1, (0.45, 0.0), 0.0, (-2.4, 0.05), 0.3),
        Joint("hip_r", 3, 0, (0.0, 0.0), math.pi, (-2.2, 1.2), 0.5),
        Joint("knee_r", 4, 3, (0.45, 0.0), 0.0, (-2.4, 0.05), 0.3),
    ]
    q0 = np.array([0.0, 0.92, math.pi / 2, 0.1, -0.2, -0.1, -0.2])
    mus = []
    for side, (th, sh) in (("l", (1, 2)), ("r", (3, 4))):
        mus += [
            make_muscle(m, f"hip_flexor_{side}", [(0, (0.12, -0.06)), (th, (0.12, -0.04))], q0, 2500.0),
            make_muscle(m, f"hip_extensor_{side}", [(0, (0.10, 0.07)), (th, (0.12, 0.04))], q0, 2500.0),
            make_muscle(m, f"knee_flexor_{side}", [(th, (0.30, 0.04)), (sh, (0.06, 0.03))], q0, 2000.0),
            make_muscle(m, f"knee_extensor_{side}", [(th, (0.30, -0.05)), (sh, (0.06, -0.035))], q0, 2000.0),
            make_muscle(m, f"hamstring_{side}", [(0, (0.05, 0.06)), (th, (0.25, 0.05)), (sh, (0.07, 0.03))], q0, 1500.0),
            make_muscle(m, f"rectus_{side}", [(0, (0.08, -0.06)), (th, (0.30, -0.06)), (sh, (0.05, -0.04))], q0, 1500.0),
            make_muscle(m, f"gastroc_{side}", [(th, (0.40, 0.04)), (sh, (0.25, 0.04)), (sh, (0.42, 0.02))], q0, 800.0),
            make_muscle(m, f"tibialis_{side}", [(th, (0.38, -0.03)), (sh, (0.20, -0.035)), (sh, (0.42, -0.02))], q0, 800.0),
        ]
    m.muscles = mus
    m.spheres = [
        {"link": 2, "offset": [0.45, 0.0], "radius": 0.04},
        {"link": 2, "offset": [0.40, -0.05], "radius": 0.03},
        {"link": 4, "offset": [0.45, 0.0], "radius": 0.04},
        {"link": 4, "offset": [0.40, -0.05], "radius": 0.03},
    ]
    m.key_bodies = [0, 2, 4]
    return m


# --------------------------------------------------------------------------
# whole-body planar humanoid: 80 links, 700 muscles
# --------------------------------------------------------------------------
def _wb_tree():
    """Returns (links, joints-with-parents-by-name) in DFS preorder."""
    nodes = []  # (name, parent_name, length, mass, anchor(local in parent), mount, limits)

    def add(name, parent, length, mass, anchor, mount, limits=(-1.5, 1.5)):
        nodes.append((name, parent, length, mass, anchor, mount, limits))

    add("pelvis", None, 0.20, 10.0, None, 0.0)
    # spine: pelvis local x = forward; spine points up (mount +pi/2)
    spine = [("L1", 0.07, 2.5), ("L2", 0.07, 2.5), ("L3", 0.07, 2.5), ("T1", 0.08, 3.0), ("T2", 0.08, 3.0),
             ("T3", 0.08, 3.0), ("T4", 0.08, 3.0), ("C1", 0.04, 0.4), ("C2", 0.04, 0.4), ("C3", 0.04, 0.4),
             ("head", 0.22, 4.5)]
    legs_and_arms_done = False
    prev = "pelvis"
    for i, (nm, ln, ms) in enumerate(spine):
        anchor = (0.0, 0.10) if prev == "pelvis" else (None, 0.0)
        mount = math.pi / 2 if prev == "pelvis" else 0.0
        add(nm, prev, ln, ms, anchor, mount, (-0.6, 0.6))
        if nm == "T2":
            for side, sgn in (("l", 1.0), ("r", -1.0)):
                add(f"clavicle_{side}", "T2", 0.06, 0.3, (None, 0.02 * sgn), -math.pi / 2, (-0.5, 0.5))
                add(f"scapula_{side}", f"clavicle_{side}", 0.06, 0.5, (None, 0.0), -math.pi / 2, (-0.6, 0.6))
                add(f"humerus_{side}", f"scapula_{side}", 0.30, 2.0, (None, 0.0), 0.0, (-2.5, 2.5))
                add(f"ulna_{side}", f"humerus_{side}", 0.26, 1.2, (None, 0.0), 0.2, (-0.2, 2.4))
                add(f"hand_{side}", f"ulna_{side}", 0.08, 0.4, (None, 0.0), 0.0, (-1.2, 1.2))
                for f, off in enumerate((-0.02, -0.01, 0.0, 0.01, 0.02)):
                    pf = f"hand_{side}"
                    for k, (fl, fm) in enumerate(((0.035, 0.08), (0.03, 0.07), (0.025, 0.06), (0.02, 0.05))):
                        cn = f"finger{f}_{k}_{side}"
                        anc = (None, off) if k == 0 else (None, 0.0)
                        add(cn, pf, fl, fm, anc, 0.0, (-0.3, 1.6))
                        pf = cn
        if nm in ("T3", "T4"):
            add(f"rib_a_{nm}", nm, 0.10, 0.5, (0.04, 0.03), -1.2, (-0.2, 0.2))
            add(f"rib_b_{nm}", nm, 0.10, 0.5, (0.04, -0.03), 1.2 - math.pi, (-0.2, 0.2))
        prev = nm
    for side in ("l", "r"):
        add(f"thigh_{side}", "pelvis", 0.42, 7.0, (0.0, -0.08), -math.pi / 2, (-1.2, 2.0))
        add(f"shank_{side}", f"thigh_{side}", 0.40, 3.0, (None, 0.0), 0.0, (-2.4, 0.05))
        add(f"talus_{side}", f"shank_{side}", 0.04, 0.3, (None, 0.0), 0.0, (-0.5, 0.5))
        add(f"calcaneus_{side}", f"talus_{side}", 0.07, 0.6, (None, 0.0), math.pi / 2, (-0.7, 0.7))
        add(f"midfoot_{side}", f"calcaneus_{side}", 0.07, 0.3, (None, 0.0), 0.0, (-0.3, 0.3))
        add(f"toes_{side}", f"midfoot_{side}", 0.04, 0.15, (None, 0.0), 0.0, (-0.5, 0.8))
        add(f"toetip_{side}", f"toes_{side}", 0.025, 0.1, (None, 0.0), 0.0, (-0.5, 0.8))
    del legs_and_arms_done
    return nodes


def _depths(model):
    fc = 1 if model.floating else 0
    d = [0] * len(model.links)
    for j, jt in enumerate(model.joints):
        d[fc + j] = (d[jt.parent] + 1) if jt.parent >= 0 else 1
    return d


def wb700(floating=True):
    name = "wb700" if floating else "wb700_fixed"
    m = Model(name, "floating" if floating else "fixed")
    m.joint_limit_stiffness = 50.0
    nodes = _wb_tree()
    # DFS preorder so that parent < child (model.cpp:37-46)
    children = {}
    for nd in nodes:
        children.setdefault(nd[1], []).append(nd)
    order = []

    def visit(nd):
        order.append(nd)
        for c in children.get(nd[0], []):
            visit(c)

    visit(nodes[0])
    index = {nd[0]: i for i, nd in enumerate(order)}
    total = sum(nd[3] for nd in order)
    scale = 60.0 / total  # PAPER.md:271 total mass 60 kg
    for nd in order:
        nm, parent, ln, ms, anchor, mount, lim = nd
        mass = ms * scale
        # radius of gyration floored at 0.1 m (synthetic armature keeps the
        # 2 ms explicit step stable for the short segments)
        m.links.append(Link(nm, ln, mass, mass * max(ln * ln / 12.0, 0.01), 0.5 * ln))
    for i, nd in enumerate(order):
        nm, parent, ln, ms, anchor, mount, lim = nd
        if parent is None:
            if not floating:
                m.joints.append(Joint("pelvis_pitch", 0, -1, (0.0, 1.0), 0.0, (-0.8, 0.8), 0.0))
            continue
        p = index[parent]
        ax = m.links[p].length if anchor[0] is None else anchor[0]
        m.joints.append(Joint(f"j_{nm}", i, p, (ax, anchor[1]), mount, lim, 0.0))
    nl = len(m.links)
    assert nl == 80, nl
    q0 = np.zeros(m.nq)
    if floating:
        q0[1] = 1.0
    # Explicit (semi-implicit Euler, 2 ms) stability is governed by the
    # *local* inertia of the links next to each joint (zig-zag modes), not
    # the subtree inertia: damping c*dt/I_loc and stiffness k*dt^2/I_loc are
    # kept well below the Euler limits (2 and 4) with these budgets.
    iloc = [joint_local_inertia(m, j, q0) for j in range(len(m.joints))]
    for j in range(len(m.joints)):
        m.joints[j].damping = round(0.05 * iloc[j] / 0.002, 9)
    # ---- muscles: 700, 2-4 via points, spanning 1-3 joints ----------------
    rng = np.random.default_rng(700)
    fc = 1 if floating else 0
    parent_of = {fc + j: jt.parent for j, jt in enumerate(m.joints)}
    joint_of_child = {fc + j: j for j in range(len(m.joints))}
    ieff = [joint_eff_inertia(m, j, q0) for j in range(len(m.joints))]

    def width(l):
        return max(0.004, 0.12 * m.links[l].length) + (0.02 if m.links[l].mass > 1.5 else 0.0)

    def point_on(l, frac, side, wscale=1.0):
        L = m.links[l].length
        return (l, (float(frac * L), float(side * width(l) * wscale)))

    # candidate chains: (joint list, link chain) of length 1..3 ending at a child link
    chains = {1: [], 2: [], 3: []}
    for c in range(nl):
        if c not in parent_of or parent_of[c] < 0:
            continue
        chain = [c]
        cur = c
        for span in (1, 2, 3):
            p = parent_of.get(cur, -1)
            if p < 0:
                break
            chain = [p] + chain
            chains[span].append(list(chain))
            cur = p
    # weights: heavier joints receive more muscles (paper's 700 are dense at hips/knees/spine)
    def chain_weight(ch):
        js = [joint_of_child[l] for l in ch[1:]]
        return sum(1.0 + 4.0 * math.sqrt(ieff[j]) for j in js)

    specs = []  # (chain, side)
    for span, count in ((1, 380), (2, 230), (3, 90)):
        cands = chains[span]
        w = np.array([chain_weight(ch) for ch in cands], dtype=float)
        w = w / w.sum()
        picks = rng.choice(len(cands), size=count, replace=True, p=w)
        for k, pi in enumerate(picks):
            specs.append((cands[pi], 1.0 if (k % 2 == 0) else -1.0))
    # every joint gets at least an agonist/antagonist pair
    have = set()
    for ch, s in specs:
        for l in ch[1:]:
            have.add((joint_of_child[l], s))
    extra = []
    for j in range(len(m.joints)):
        c = fc + j
        if parent_of[c] < 0:
            continue
        for s in (1.0, -1.0):
            if (j, s) not in have:
                extra.append(([parent_of[c], c], s))
    n_world = 0 if floating else 4
    specs = extra + specs[: 700 - n_world - len(extra)]
    assert len(specs) == 700 - n_world

    # per-joint muscle counts for the force scaling
    per_joint = [0] * len(m.joints)
    for ch, s in specs:
        for l in ch[1:]:
            per_joint[joint_of_child[l]] += 1

    mus = []
    for idx, (ch, side) in enumerate(specs):
        vps = [point_on(ch[0], rng.uniform(0.35, 0.85), side, rng.uniform(0.6, 1.2))]
        for l in ch[1:-1]:
            vps.append(point_on(l, rng.uniform(0.3, 0.7), side, rng.uniform(0.8, 1.4)))
        vps.append(point_on(ch[-1], rng.uniform(0.15, 0.45), side, rng.uniform(0.5, 1.0)))
        # f_max sized so each joint's summed Hill damping (dF/dv at v=0 is
        # 1.25 f_max / (l_opt v_max)) stays at c*dt/I_loc <= 0.3
        js = [joint_of_child[l] for l in ch[1:]]
        origin, angle, _ = fk(m, q0)
        L = mtu_len(m, origin, angle, vps)
        l_opt = 0.6 * L
        arms = moment_arms_fd(m, vps, q0, js)
        cap = min(0.3 * iloc[j] * l_opt * 10.0 / (max(r, 1e-3) ** 2 * 1.25 * 0.002 * per_joint[j])
                  for j, r in zip(js, arms))
        f_max = float(min(3000.0, cap))
        tau_act = float(rng.uniform(0.008, 0.012))
        tau_deact = float(rng.uniform(0.035, 0.045))
        nm = "m%03d_%s_%s" % (idx, m.links[ch[0]].name, m.links[ch[-1]].name)
        mus.append(make_muscle(m, nm, vps, q0, round(f_max, 6), 10.0, tau_act, tau_deact))
    for k in range(n_world):  # pinned pelvis: world-anchored pitch actuators
        side = 1.0 if k % 2 == 0 else -1.0
        vps = [(-1, (0.15 * side, 1.0 + 0.05 * (k // 2))), (0, (0.1 * side, 0.06 * side))]
        mus.append(make_muscle(m, "pelvis_world_%d" % k, vps, q0, 3000.0))
    m.muscles = mus

    # key bodies (PAPER.md:279 xpos in R^30 -> 10 bodies)
    kb = ["pelvis", "T4", "head", "hand_l", "hand_r", "calcaneus_l", "calcaneus_r", "shank_l", "shank_r", "ulna_l"]
    m.key_bodies = [index[n] for n in kb]
    if floating:
        m.contact = {"stiffness": 2.0e4, "damping": 120.0, "friction": 0.9, "smoothing_vel": 0.05}
        sp = []
        for side in ("l", "r"):
            sp.append({"link": index[f"calcaneus_{side}"], "offset": [0.0, -0.01], "radius": 0.025})
            sp.append({"link": index[f"midfoot_{side}"], "offset": [0.07, -0.01], "radius": 0.02})
            sp.append({"link": index[f"toetip_{side}"], "offset": [0.025, 0.0], "radius": 0.015})
            sp.append({"link": index[f"hand_{side}"], "offset": [0.04, 0.0], "radius": 0.02})
            sp.append({"link": index[f"finger2_3_{side}"], "offset": [0.02, 0.0], "radius": 0.01})
        m.spheres = sp
    return m


# --------------------------------------------------------------------------
# clips
# --------------------------------------------------------------------------
def finite_diff(q, dt):
    dq = np.zeros_like(q)
    dq[1:-1] = (q[2:] - q[:-2]) / (2 * dt)
    dq[0] = (q[1] - q[0]) / dt
    dq[-1] = (q[-1] - q[-2]) / dt
    return dq


def clip_rows(model: Model, q):
    T = q.shape[0]
    dq = finite_diff(q, CTRL_DT)
    nk = len(model.key_bodies)
    kp = np.zeros((T, 2 * nk))
    ka = np.zeros((T, nk))
    for t in range(T):
        origin, angle, _ = fk(model, q[t])
        pos, ang = key_body_state(model, origin, angle)
        for k in range(nk):
            kp[t, 2 * k] = pos[k][0]
            kp[t, 2 * k + 1] = pos[k][1]
            ka[t, k] = ang[k]
    return dq, kp, ka


def write_clip(path, model: Model, q):
    dq, kp, ka = clip_rows(model, q)
    T = q.shape[0]
    nq = model.nq
    nk = len(model.key_bodies)
    cols = ["time"] + [f"q_{j}" for j in range(nq)] + [f"dq_{j}" for j in range(nq)]
    for k in range(nk):
        cols += [f"key{k}_x", f"key{k}_z"]
    cols += [f"key{k}_angle" for k in range(nk)]
    with open(path, "w") as f:
        f.write(",".join(cols) + "\n")
        for r in range(T):
            row = [r / RATE] + list(q[r]) + list(dq[r]) + list(kp[r]) + list(ka[r])
            f.write(",".join("%.17g" % v for v in row) + "\n")


def sinusoid_clip(model: Model, T, seed):
    """Low-pass filtered multi-sine around the neutral pose (small models)."""
    rng = np.random.default_rng(seed)
    t = np.arange(T) / RATE
    q = np.zeros((T, model.nq))
    if model.floating:
        q[:, 0] = 0.3 * t / t[-1]
        q[:, 1] = 0.92 + 0.01 * np.sin(2 * np.pi * 1.0 * t)
        q[:, 2] = math.pi / 2 + 0.05 * np.sin(2 * np.pi * 0.5 * t)
    for j in range(len(model.joints)):
        d = model.nrd + j
        lo, hi = model.joints[j].limits
        mid = 0.5 * (lo + hi) if hi - lo < 3.0 else 0.0
        amp = min(0.5, 0.3 * (hi - lo))
        f1, f2 = rng.uniform(0.3, 0.8), rng.uniform(0.8, 1.5)
        ph1, ph2 = rng.uniform(0, 2 * np.pi, size=2)
        q[:, d] = mid + amp * (0.7 * np.sin(2 * np.pi * f1 * t + ph1) + 0.3 * np.sin(2 * np.pi * f2 * t + ph2))
    return q


def dance_clip(model: Model, T, seed=11):
    """Multi-sine joint trajectories, 0.2-0.6 rad at 0.5-2 Hz, plus root drift."""
    rng = np.random.default_rng(seed)
    t = np.arange(T) / RATE
    q = np.zeros((T, model.nq))
    if model.floating:
        q[:, 0] = 0.15 * np.sin(2 * np.pi * 0.1 * t)
        q[:, 1] = 1.0 + 0.03 * np.sin(2 * np.pi * 1.0 * t)
        q[:, 2] = 0.1 * np.sin(2 * np.pi * 0.25 * t)
    for j in range(len(model.joints)):
        d = model.nrd + j
        lo, hi = model.joints[j].limits
        mid = 0.5 * (lo + hi)
        half = 0.5 * (hi - lo)
        amp = min(rng.uniform(0.2, 0.6), 0.8 * half)
        f = rng.uniform(0.5, 2.0)
        ph = rng.uniform(0, 2 * np.pi)
        q[:, d] = mid + amp * np.sin(2 * np.pi * f * t + ph) * (0.6 + 0.4 * np.sin(2 * np.pi * 0.05 * t))
    return q


def backflip_clip(model: Model, T, seed=13):
    """Root pitch ramps through -2*pi in 1 s with a parabolic root height and
    tucked hips/knees; one flip every 2.5 s (exercises wrap_angle)."""
    assert model.floating
    rng = np.random.default_rng(seed)
    t = np.arange(T) / RATE
    q = np.zeros((T, model.nq))
    period, flip = 2.5, 1.0
    ph = np.mod(t, period)
    n_done = np.floor(t / period)
    in_flip = ph < flip
    s = np.clip(ph / flip, 0.0, 1.0)
    q[:, 0] = 0.05 * t
    q[:, 1] = 1.0 + np.where(in_flip, 4.0 * 0.6 * s * (1.0 - s), 0.0)
    smooth = s * s * (3.0 - 2.0 * s)
    q[:, 2] = -2.0 * np.pi * (n_done + np.where(in_flip, smooth, 1.0))
    tuck = np.where(in_flip, np.sin(np.pi * s), 0.0)
    for j, jt in enumerate(model.joints):
        d = model.nrd + j
        nm = jt.name
        lo, hi = jt.limits
        base = 0.05 * np.sin(2 * np.pi * rng.uniform(0.3, 1.0) * t + rng.uniform(0, 6.28))
        if nm.startswith("j_thigh"):
            q[:, d] = base + 1.4 * tuck
        elif nm.startswith("j_shank"):
            q[:, d] = base - 1.6 * tuck
        else:
            q[:, d] = np.clip(base, lo, hi)
    return q


# --------------------------------------------------------------------------
def wb700_general():
    """wb700_fixed with every multi-joint muscle's interior via points removed:
    its single segment then joins two links that are NOT parent and child (a
    straight bi-/tri-articular line of action), which the device evaluates on
    its generic world-frame path (general segments + per-joint pairs,
    skeleton.cpp:147-170) instead of the adjacent-segment fast path.  l_opt is
    kept and the tendon slack reset so each fibre is at its optimal length in
    the neutral pose.  Uses the wb700_fixed clip (same tree and key bodies)."""
    m = wb700(False)
    m.name = "wb700_general"
    q0 = np.zeros(m.nq)
    origin, angle, _ = fk(m, q0)
    for mu in m.muscles:
        vps = mu["via_points"]
        if len(vps) < 3:
            continue
        keep = [vps[0], vps[-1]]
        L = mtu_len(m, origin, angle, [(v[0], tuple(v[1])) for v in keep])
        mu["via_points"] = keep
        mu["tendon_slack"] = float(max(0.0, L - mu["l_opt"]))
    return m


def wb700_slow():
    """BASELINE c5 stress model: wb700 (floating, contacts) with a long
    excitation-to-activation lag on every muscle, tau_act = 0.05 s and
    tau_deact = 0.20 s (the reference has no transport delay; the first-order
    activation lag is its only delay, muscle.cpp:42-56).  Clip: wb700_dance."""
    m = wb700(True)
    m.name = "wb700_slow"
    for mu in m.muscles:
        mu["tau_act"], mu["tau_deact"] = 0.05, 0.20
    return m


def write_model(path, model):
    with open(path, "w") as f:
        json.dump(model.to_json(), f, indent=1)


def generate(out_dir, which=None):
    os.makedirs(out_dir, exist_ok=True)
    jobs = {
        "pendulum1_m2": (pendulum1_m2, [("sine", lambda m: sinusoid_clip(m, 1101, 1))]),
        "arm2_m6": (arm2_m6, [("sine", lambda m: sinusoid_clip(m, 1101, 2))]),
        "walker5_m16": (walker5_m16, [("sine", lambda m: sinusoid_clip(m, 1101, 3))]),
        "wb700": (lambda: wb700(True), [("dance", lambda m: dance_clip(m, 1101)),
                                         ("backflip", lambda m: backflip_clip(m, 1101))]),
        "wb700_fixed": (lambda: wb700(False), [("dance", lambda m: dance_clip(m, 1101))]),
        "wb700_general": (wb700_general, []),  # clip: wb700_fixed_dance (same tree)
        "wb700_slow": (wb700_slow, []),  # clip: wb700_dance (same tree)
    }
    written = []
    for name, (mk, clips) in jobs.items():
        if which and name not in which:
            continue
        model = mk()
        mp = os.path.join(out_dir, f"{name}.json")
        write_model(mp, model)
        written.append(mp)
        for cname, fn in clips:
            cp = os.path.join(out_dir, f"{name}_{cname}.csv")
            write_clip(cp, model, ground_offset(model, fn(model)))
            written.append(cp)
    return written


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "assets", "generated"))
    ap.add_argument("models", nargs="*")
    a = ap.parse_args()
    for p in generate(a.out, a.models or None):
        print(p)


if __name__ == "__main__":
    main()
