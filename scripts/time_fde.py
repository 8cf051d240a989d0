"""Full-domain evaluation (ogm_fss_full_domain) at the C1 / C3 / C4 key-batch
shapes, checked against the first run: python scripts/time_fde.py."""
import sys, os
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2209_03526_b200 import _lib, fss
_lib.check(_lib.load().ogm_init())
rng = np.random.default_rng(3)
for comparison, nkeys, bits, n in ((True, 12, 14, 10000), (False, 6, 14, 10000), (True, 12, 18, 182083), (True, 6, 9, 333), (False, 6, 10, 1000)):
    alphas = rng.integers(0, n, size=nkeys, dtype=np.uint64)
    r0 = rng.integers(0, 256, (nkeys, 16), dtype=np.uint8); r1 = rng.integers(0, 256, (nkeys, 16), dtype=np.uint8)
    dev = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).view(dt).cuda()
    b0, _ = fss.gen_batch(comparison, bits, dev(alphas.astype(np.uint32), torch.int32), dev(r0, torch.uint8), dev(r1, torch.uint8))
    ref = fss.full_domain(b0, n).clone()
    for _ in range(3): fss.full_domain(b0, n)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(20): out = fss.full_domain(b0, n)
    b.record(); torch.cuda.synchronize()
    print(os.environ.get("OGM_FDE_KK", "auto"), "DCF" if comparison else "DPF", nkeys, bits, n, round(a.elapsed_time(b) / 20 * 1e3, 1), "us", bool(torch.equal(out, ref)), flush=True)
