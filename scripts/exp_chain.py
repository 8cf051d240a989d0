"""Chained planned online shuffle (ogm_shuffle_online_planned_ex: each message
handed sender -> receiver in shared memory) vs the four planned party steps,
at 2^lg rows x 128 bits.  Checks x1, y1, c1, R3 against the step-wise path,
then times: steps (output-order blinds), steps with source-order blinds, the
chained kernel with and without message copies.  L2 flushed between
iterations below 4x L2."""
import statistics
import sys

sys.path.insert(0, ".")
import torch

from paper_2209_03526_b200 import _lib, workloads
from paper_2209_03526_b200.net import make_session_configs
from paper_2209_03526_b200.shuffle import ShuffleOffline, source_order

_lib.check(_lib.load().ogm_init())
flush = torch.empty((512 << 20,), dtype=torch.uint8, device="cuda")
P = _lib.ptr


def arr(ts, ctype):
    import ctypes
    return (ctype * len(ts))(*[P(t) for t in ts])


for lg in map(int, sys.argv[1:]):
    import ctypes
    rows = 1 << lg
    cfg = make_session_configs(b"\x77" * 16)
    comps = [workloads.device_random_words(rows * 4, 1, 20 + c).reshape(rows, 4) for c in range(3)]
    e = lambda: torch.empty_like(comps[0])  # noqa: E731
    off = [ShuffleOffline(p + 1, cfg[p].seed_with_next, cfg[p].seed_with_prev, 0, rows, 128, plan=True)
           for p in range(3)]
    # the blinds as the chained shuffle expects them (W in c1's output order above 256 MB)
    (u_src,), (v_src, w_src), (z_src,) = (o.chain_blinds("slot") for o in off)
    w_steps = source_order(off[1].w, off[1].pi23)   # the per-party steps with source-order blinds
    plans = [off[0].plan_x1, off[1].plan_y1, off[1].plan_c1, off[2].plan_r3]
    want = [e() for _ in range(4)]
    off[0].step_x1(comps[0], comps[1], want[0])
    off[1].step_y1(comps[2], want[1])
    off[1].step_c1(want[0], want[2])
    off[2].step_r3(want[1], want[2], want[3])
    inter = [e() for _ in range(3)]
    got = [e() for _ in range(4)]
    q2 = (ctypes.c_void_p * 4)(*[P(p.q2) for p in plans])
    gd = (ctypes.c_void_p * 4)(*[P(p.gdst) for p in plans])
    sr = (ctypes.c_void_p * 4)(*[P(p.srow) for p in plans])
    it = (ctypes.c_void_p * 3)(*[P(t) for t in inter])

    def chained(msgs: bool):
        # chain_blinds("slot"): U', V' in source order, W and Z in slot order (W in output order above 256 MB)
        _lib.call("ogm_shuffle_online_planned_ex", rows, ctypes.addressof(q2), ctypes.addressof(gd),
                  ctypes.addressof(sr), P(comps[0]), P(comps[1]), P(comps[2]), P(u_src), P(v_src), 0, P(w_src),
                  1 if off[1].w_output_order else 2, P(z_src), 2, ctypes.addressof(it),
                  P(got[0]) if msgs else None, P(got[1]) if msgs else None, P(got[2]) if msgs else None,
                  P(got[3]), _lib.stream_ptr())

    chained(True)
    torch.cuda.synchronize()
    ok = [bool(torch.equal(g, w)) for g, w in zip(got, want)]
    got[3].zero_()
    chained(False)
    ok.append(bool(torch.equal(got[3], want[3])))
    x1, y1, c1, r3 = (e() for _ in range(4))
    sink = e()

    def steps():
        off[0].step_x1(comps[0], comps[1], x1)
        off[1].step_y1(comps[2], y1)
        off[1].step_c1(x1, c1)
        off[2].step_r3(y1, c1, r3)

    def steps_src():
        plans[0].run(x1, m1=comps[0], m2=comps[1], m4=u_src)
        plans[1].run(y1, m1=comps[2], m4=v_src)
        plans[2].run(c1, m1=x1, m4=w_steps)
        plans[3].run(r3, m1=y1, m3=c1, m4=z_src)

    steps_src()
    ok.append(bool(torch.equal(r3, want[3])))
    res = {}
    small = rows * 16 * 4 < (512 << 20)
    for name, fn in (("steps", steps), ("steps_src", steps_src), ("chain_msgs", lambda: chained(True)),
                     ("chain", lambda: chained(False))):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(7):
            if small:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res[name] = statistics.median(ts)
    print(f"2^{lg} equal={ok}: " + "  ".join(f"{k} {v:.4f} ms ({240 * rows / (v * 1e-3) / 1e9 / 6535:.3f})"
                                            for k, v in res.items()), flush=True)
    del off, plans, want, inter, got, comps, u_src, v_src, w_src, z_src, w_steps, x1, y1, c1, r3, sink
    torch.cuda.empty_cache()
