"""Dump full device states of a few propagations to an .npz, to compare two
builds of the library bit for bit (e.g. the element-parallel kernel against
k_mm4):  HEOM_B200_LIB=... python tools/bitwise_dump.py out.npz
         python tools/bitwise_dump.py --compare a.npz b.npz"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

if sys.argv[1] == "--compare":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    ok = True
    for k in a.files:
        same = np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8))
        diff = float(np.max(np.abs(a[k] - b[k]))) if not same else 0.0
        print(f"{k}: {'bit-identical' if same else 'DIFFERENT max|d| = %.3e' % diff}")
        ok = ok and same
    sys.exit(0 if ok else 1)

import paper_1012_4382_b200 as xf  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_1012_4382_b200.engine import BlockOperands, DeviceRun  # noqa: E402
from tests.cases import BATH300, FMO, RATES  # noqa: E402
from tests.test_gpu_fullstate import random_hermitian_hierarchy  # noqa: E402

out = {}
for K, n_max, steps, order in [(0, 3, 10, "reference"), (1, 4, 10, "reference"), (1, 4, 10, "lex"),
                               (0, 6, 200, "reference"), (1, 8, 3, "reference")]:
    tiers = orc.enumerate_hierarchy(7 * (K + 1), n_max)[1]
    sig0 = random_hermitian_hierarchy(tiers, 7, seed=1 + K + n_max)
    ops = BlockOperands(FMO, BATH300, RATES, K)
    with DeviceRun(ops, n_max, 1.0, t_end_fs=float(steps), ordering=order, record_stride=1) as run:
        run.set_state(sig0, [0.0, 0.0])
        run.run()
        sig, sinks = run.state(sig0.shape[0])
        _, pops, _ = run.records()
    key = f"K{K}_N{n_max}_{steps}_{order}"
    out[key + "_state"] = sig
    out[key + "_pops"] = pops
    out[key + "_sinks"] = sinks
np.savez(sys.argv[1], **out)
print("wrote", sys.argv[1])
