"""The trio masked parity (ogm_masked_parity, all three parties) at the C3 /
C4 attribute shapes, one pass (a folded interval or an equality) against two:
python scripts/time_masked_parity.py."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2209_03526_b200 import _lib, workloads
A = _lib.ptr_array
_lib.check(_lib.load().ogm_init())
for rows, words in ((200_000, 5691), (2_000_000, 313), (200_000, 2000)):
    pitch = (words + 3) // 4 * 4
    comps = [workloads.device_random_words(rows * pitch, 1, 10 + c).reshape(rows, pitch) for c in range(3)]
    inds = [workloads.device_random_words(pitch, 2, 20 + j)[:words] for j in range(12)]
    for npass in (1, 2):
        outs = [torch.empty(((rows + 31) // 32,), dtype=torch.int32, device="cuda") for _ in range(3 * npass)]
        f = lambda: _lib.call("ogm_masked_parity", rows, words, pitch, 3, A(comps), 3, _lib.int_array([0, 1, 2]),
                              _lib.int_array([1, 2, 0]), npass, A(inds[:6 * npass]), A(outs), _lib.stream_ptr())
        for _ in range(3): f()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        for _ in range(10): f()
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        print(rows, words, npass, round(ms, 4), "ms", round(3 * rows * words * 4 / ms / 1e9, 1), "TB/s", flush=True)
