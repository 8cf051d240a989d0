"""C5 at 2^lg through ShuffleOffline (the bench's allocation state), per-pass events."""
import sys

sys.path.insert(0, ".")
import torch

from paper_2209_03526_b200 import _lib, workloads
from paper_2209_03526_b200.net import make_session_configs
from paper_2209_03526_b200.prf import seeded_permutation_device
from paper_2209_03526_b200.shuffle import ShuffleOffline

_lib.check(_lib.load().ogm_init())
rows = 1 << int(sys.argv[1])
cfg = make_session_configs(b"\x77" * 16)
comps = [workloads.device_random_words(rows * 4, 1, 20 + c).reshape(rows, 4) for c in range(3)]
pc = {}
off = [ShuffleOffline(p + 1, cfg[p].seed_with_next, cfg[p].seed_with_prev, 0, rows, 128, perm_cache=pc)
       for p in range(3)]
x1, y1, c1, r3 = (torch.empty_like(comps[0]) for _ in range(4))
print(f"allocated {torch.cuda.memory_allocated() / 2**30:.1f} GiB, reserved {torch.cuda.memory_reserved() / 2**30:.1f}")
steps = [(off[0].plan_x1, dict(m1=comps[0], m2=comps[1], r=off[0].u), x1),
         (off[1].plan_y1, dict(m1=comps[2], r=off[1].v), y1),
         (off[1].plan_c1, dict(m1=x1, r=off[1].w), c1),
         (off[2].plan_r3, dict(m1=y1, m3=c1, m4=off[2].z), r3)]
for rep in range(3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(9)]
    ev[0].record()
    for k, (pl, kw, out) in enumerate(steps):
        it = torch.empty_like(comps[0])
        pl.run(out, inter=it, passes=1, **kw)
        ev[2 * k + 1].record()
        pl.run(out, inter=it, passes=2, **kw)
        ev[2 * k + 2].record()
        del it
    torch.cuda.synchronize()
    print([round(ev[i].elapsed_time(ev[i + 1]), 3) for i in range(8)])
