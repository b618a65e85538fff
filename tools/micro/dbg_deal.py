import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle as O
from paper_2402_02320_b200.mpfix.preprocessing import DemandCounter, memory_stores
from paper_2402_02320_b200.mpfix.session import PartySession
from paper_2402_02320_b200.mpfix.metrics import CommMetrics
from paper_2402_02320_b200.mpfix.transport import NullMesh
import test_acceptance_b200 as A
import test_dealer_fused as T
for n in (2, 3):
    counter = DemandCounter(party=0)
    A._protocol_batch(PartySession(0, n, NullMesh(0, n), counter, metrics=CommMetrics(0, n)))
    dem = dict(counter.demands)
    stores = memory_stores(11, n, dem)
    torch.cuda.synchronize()
    for key, count in dem.items():
        want = O.deal_material(11, n, key.name(), count)
        for p in range(n):
            got = stores[p]._arrays[key]
            for arr, w in want.items():
                g = T._as_np(got[arr], w[p:p + 1])
                if not np.array_equal(g, w[p:p + 1]):
                    bad = np.argwhere(g.reshape(-1) != w[p:p+1].reshape(-1))
                    print("MISMATCH", n, key.name(), p, arr, bad.size, bad[:3].ravel())
    print("done", n)
