import sys; sys.path.insert(0, '.')
import numpy as np
from oracle import oracle as orc
from paper_1012_4382_b200.engine import BlockOperands, DeviceRun
from tests.cases import BATH300, FMO, RATES
from tests.test_gpu_fullstate import random_hermitian_hierarchy, _oracle_state
K, n = 0, 1
tiers = orc.enumerate_hierarchy(7, n)[1]
full = random_hermitian_hierarchy(tiers, 7, 5)
ops = BlockOperands(FMO, BATH300, RATES, K)
for name, mask in (("ado0 only", tiers == 0), ("tier1 only", tiers == 1), ("ado 1 only", np.arange(8) == 1), ("ado 7 only", np.arange(8) == 7)):
    sig0 = full * mask[:, None, None]
    ref = _oracle_state(K, n, 1, sig0)["final_state"]
    with DeviceRun(ops, n, 1.0, t_end_fs=1e9, record_stride=1) as run:
        run.set_state(sig0, [0.0, 0.0])
        run.time_steps(1)
        st, _ = run.state(len(tiers))
    d = np.abs(st - ref)
    print(name, "per-ADO max err", np.round(d.max(axis=(1, 2)), 6))
    k = int(np.argmax(d.max(axis=(1, 2))))
    print("   worst ADO", k, "err matrix rows (abs):")
    print(np.round(d[k], 4))
