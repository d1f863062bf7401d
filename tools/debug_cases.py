"""Run each golden engine case in its own process (GPU box debugging aid).

    RBC_DEBUG_SYNC=1 python tools/debug_cases.py [dense|plan|leaf]
"""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

CHILD = r"""
import sys, json, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + '/tests')
from conftest import case_levels, mode_for, same_values
from paper_1905_07439_b200 import engine
from paper_1905_07439_b200._lib import FORMULA_IDS
meta = json.load(open({root!r} + '/tests/golden/engine_cases.json'))
arrs = np.load({root!r} + '/tests/golden/engine_cases.npz')
kind, name = {kind!r}, {name!r}
if kind == 'leaf':
    case = [c for c in meta['leaf'] if c['name'] == name][0]
    out = engine.leaf_matmul(arrs[name + '/x'], arrs[name + '/y'], mode_for(case['mode']))
    print('OK' if same_values(out, arrs[name + '/out']) else 'MISMATCH')
    sys.exit(0)
case = [c for c in meta['engine'] if c['name'] == name][0]
mode = mode_for(case['mode'])
a, b = arrs[name + '/a'], arrs[name + '/b']
try:
    if kind == 'dense':
        out = engine.apply_levels(case_levels(arrs, name, case['Q']), a, b, mode)
    else:
        Q, n = case['Q'], case['n']
        p, s = arrs[name + '/perms'], arrs[name + '/signs']
        packed = engine.pack_plans(n, p.reshape(-1, 3, n), s.reshape(-1, 3, n)).reshape(p.shape[0], Q, -1)
        out = engine.apply_plans(FORMULA_IDS[case['plan_formula']], Q, packed, a, b, mode)
except OverflowError:
    print('OK (overflow)' if case['raises'] else 'UNEXPECTED OVERFLOW'); sys.exit(0)
if case['raises']:
    print('MISSED OVERFLOW'); sys.exit(0)
print('OK' if same_values(out, arrs[name + '/out']) else 'MISMATCH')
"""


def main():
    kinds = sys.argv[1:] or ["dense", "plan", "leaf"]
    meta = json.loads((ROOT / "tests/golden/engine_cases.json").read_text())
    for kind in kinds:
        if kind == "leaf":
            names = [c["name"] for c in meta["leaf"]]
        elif kind == "plan":
            names = [c["name"] for c in meta["engine"] if c["plan_formula"] and c["layout"] != "raw"]
        else:
            names = [c["name"] for c in meta["engine"]]
        for name in names:
            res = subprocess.run([sys.executable, "-c", CHILD.format(root=str(ROOT), kind=kind, name=name)],
                                 capture_output=True, text=True, timeout=300)
            line = res.stdout.strip().splitlines()[-1] if res.stdout.strip() else ""
            if res.returncode != 0:
                line = "ERROR " + (res.stderr.strip().splitlines()[-1] if res.stderr.strip() else "")
            print(f"{kind:5s} {name:32s} {line}", flush=True)


if __name__ == "__main__":
    main()
