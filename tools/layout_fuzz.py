"""Forced sweep layouts (item size / nodes per item / slot size / staging) on
small trees, each case in a subprocess, checked against the CPU oracle:
python tools/layout_fuzz.py   (prints OK / FAIL <gap> / CRASH per case)"""
import itertools
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, os, sys
import numpy as np
sys.path.insert(0, %r)
import paper_2107_01745_b200 as so
from oracle import oracle as orc
nx, nu, N, br = json.loads(sys.argv[1])
prob = so.gen_random_instance(3, nx, nu, N, br)
cache = so.factor(prob)
info = cache.dev_info()
print(json.dumps({k: info[k] for k in ("slots", "slot_bytes", "nodes_per_item_max", "items_global", "consumer_stage",
                                       "items_bw", "items_fw", "grid_ctas", "cut_stage")}), file=sys.stderr, flush=True)
ofac = orc.Factor(orc.Problem.from_flat(prob.flat()))
rng = np.random.default_rng(5)
y, r = rng.uniform(-1, 1, prob.dual_dim), rng.uniform(-1, 1, prob.dual_dim)
gap = 0.0
for affine in (True, False):
    pts, hs = so.sweep(cache, [y, r], affine)
    for v, pt in ((y, pts[0]), (r, pts[1])):
        ox, ou = ofac.sweep(v, affine)
        s = 1 + max(np.abs(ox).max(), np.abs(ou).max())
        gap = max(gap, np.abs(pt.x.ravel(order="F") - ox).max() / s, np.abs(pt.u.ravel(order="F") - ou).max() / s)
print(json.dumps(dict(gap=gap, slots=info["slots"], slot=info["slot_bytes"], npi=info["nodes_per_item_max"],
                      glob=info["items_global"], cons=info["consumer_stage"])))
''' % ROOT
shapes = [(10, 5, 9, [2] * 7), (10, 5, 8, [4, 4, 4]), (6, 3, 7, [3, 3, 2, 2]), (12, 4, 6, [2] * 6)]
knobs = [dict(SCENOPT_ITEM_KB=kb, SCENOPT_ITEM_MAX_NODES=mn, **({"SCENOPT_SLOT_KB": sk} if sk else {}),
              **({"SCENOPT_STAGE": "consumer"} if cons else {}))
         for kb, mn, sk, cons in itertools.product([24, 48, 96], [32, 64, 128], [0, 4, 16], [False, True])]
if os.environ.get("FUZZ_SET") == "extremes":  # default knobs, extreme shapes
    shapes = [(1, 1, 8, [2] * 8), (2, 1, 6, [8, 8]), (1, 2, 5, [16, 4]), (3, 1, 12, [2] * 4), (4, 4, 3, [32, 2]),
              (2, 2, 10, [3] * 6), (5, 1, 4, [64]), (8, 8, 2, [50]), (1, 1, 20, [2, 2]), (16, 2, 4, [6, 6, 2]),
              (30, 30, 3, [4, 2]), (64, 8, 3, [3, 3])]
    knobs = [{}, {"SCENOPT_GRID": 7, "SCENOPT_MIN_SUBTREES": 1}, {"SCENOPT_GRID": 148, "SCENOPT_MIN_SUBTREES": 1}]
if len(sys.argv) > 1:  # focused rerun: python tools/layout_fuzz.py SHAPE_JSON KNOBS_JSON
    shapes, knobs = [tuple(json.loads(sys.argv[1]))], [json.loads(sys.argv[2])]
for shape in shapes:
    for kn in knobs:
        env = dict(os.environ, **{k: str(v) for k, v in kn.items()})
        try:
            p = subprocess.run([sys.executable, "-c", CHILD, json.dumps(shape)], env=env, capture_output=True,
                               text=True, timeout=120)
        except subprocess.TimeoutExpired:
            print("HANG ", shape, kn, flush=True)
            continue
        if p.returncode != 0:
            err = p.stderr.strip().splitlines()
            print("CRASH", shape, kn, err[-1][:120], "| layout", next((l for l in err if l.startswith("{")), ""),
                  flush=True)
            continue
        res = json.loads(p.stdout.strip().splitlines()[-1])
        print("OK   " if res["gap"] < 1e-9 else "FAIL ", shape, kn, res, flush=True)
