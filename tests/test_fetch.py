"""The C5 fetch: sec_fetch_multi of flag + 128-bit id rows (src/engine.py:
220-270), shuffle -> open the flag column -> keep the flagged rows.

* CPU: the oracle restatement (oracle.fetch_multi_trio) against the live
  reference's recorded runs (tests/golden/c5fetch.npz, make_golden.py).
* GPU: the flag-split fetch (fetch.FlaggedFetch, the C5 bench path) against
  the oracle at up to 2^20 rows on both shuffle executions, the Trio API on
  the golden, and the per-party drop-in path against the split path.
"""

import hashlib

import numpy as np
import pytest

import oracle


def _seeds(master: bytes):
    """src/net.py:221-233 pair seeds (s12, s23, s31)."""
    d = lambda s: hashlib.sha256(master + b"/" + s.encode()).digest()[:16]  # noqa: E731
    return d("pair-seed-12"), d("pair-seed-23"), d("pair-seed-31")


def _case(g, tag):
    rows = int(g[f"{tag}_rows"])
    master = g[f"{tag}_master"].tobytes()
    ids = [g[f"{tag}_id{c}"] for c in range(3)]
    flags = [g[f"{tag}_flag{c}"] for c in range(3)]
    return rows, master, ids, flags


@pytest.mark.parametrize("n", [0, 1, 31, 32, 33, 1000, (1 << 22) + 5])
def test_bit_gather_matches_numpy(n):
    """fetch.bit_gather (offline composition of the flag blinds): bit i of
    the output = bit idx[i] of the source column, clean tail."""
    import torch

    from paper_2209_03526_b200.fetch import bit_gather

    rng = np.random.default_rng(n)
    src = rng.integers(0, 2, n, dtype=np.uint8)
    idx = rng.permutation(n).astype(np.int32)
    col = torch.from_numpy(oracle.pack_bits(src).view(np.int32).copy())
    got = bit_gather(col, torch.from_numpy(idx), n).numpy().view(np.uint32)
    want = oracle.pack_bits(src[idx])
    assert np.array_equal(got[:want.size], want)


def test_oracle_fetch_matches_reference(golden):
    g = golden("c5fetch")
    for tag in g["cases"]:
        rows, master, ids, flags = _case(g, tag)
        keep, plain, recs = oracle.fetch_multi_trio(*_seeds(master), 0, flags, ids, 128)
        for q in range(3):
            assert np.array_equal(plain, g[f"{tag}_audit{q}"]), tag
            assert int(g[f"{tag}_n{q}"]) == keep.size
            assert np.array_equal(recs[q], g[f"{tag}_ida{q}"].reshape(-1, 4)), (tag, q)
            assert np.array_equal(recs[(q + 1) % 3], g[f"{tag}_idb{q}"].reshape(-1, 4)), (tag, q)


# ---------------------------------------------------------------------------
# GPU
# ---------------------------------------------------------------------------


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32).copy()).cuda()


def _inputs(rows: int, p: float, seed: int):
    rng = np.random.default_rng(seed)
    ids = [rng.integers(0, 1 << 32, size=(rows, 4), dtype=np.uint32) for _ in range(3)]
    plain = (rng.random(rows) < p).astype(np.uint8)
    f1 = oracle.pack_bits(rng.integers(0, 2, rows, dtype=np.uint8))
    f2 = oracle.pack_bits(rng.integers(0, 2, rows, dtype=np.uint8))
    f3 = oracle.pack_bits(plain) ^ f1 ^ f2
    return ids, [f1, f2, f3], plain


@pytest.mark.gpu
@pytest.mark.parametrize("rows,p,plan,tail", [(1, 1.0, False, None), (33, 0.5, False, None),
                                              (1000, 0.1, False, None), (1 << 20, 0.1, False, None),
                                              ((1 << 20) + 77, 0.2, False, None), (1 << 21, 0.05, False, None),
                                              (1 << 20, 0.01, True, None), ((1 << 20) + 77, 1.0, True, None),
                                              (40000, 0.0, True, None), ((1 << 20) + 77, 0.3, True, True),
                                              (1 << 22, 0.1, True, True), ((1 << 24) + 33, 0.05, None, None)])
def test_flagged_fetch_matches_oracle(rows, p, plan, tail):
    """Records, opened flags and the three new components of the split
    fetch equal the oracle's sec_fetch_multi bit for bit: one cooperative
    launch, the chained shuffle + flag kernels, and the flag column riding
    the final window passes (dual pass; split passes above 256 MB)."""
    import torch

    from paper_2209_03526_b200.fetch import FlaggedFetch

    seeds = _seeds(bytes([0x5f, rows & 0xFF]) * 8)
    ids, flags, plain = _inputs(rows, p, rows)
    ff = FlaggedFetch(seeds, 3, rows, plan=plan, flag_tail=tail)
    if rows > (1 << 24):
        assert ff.flag_tail   # the split final window passes carry the flag column
    ff.online([_dev(f) for f in flags], [_dev(m) for m in ids])
    keep, want_plain, want = oracle.fetch_multi_trio(*seeds, 3, flags, ids, 128)
    got_plain = oracle.unpack_bits(ff.plain.cpu().numpy().view(np.uint32), rows)
    assert np.array_equal(got_plain, want_plain)
    recs = ff.records()
    assert recs[0].shape[0] == keep.size == int(want_plain.sum())
    for c in range(3):
        assert np.array_equal(recs[c].cpu().numpy().view(np.uint32), want[c]), c
    # the shuffled table itself: R_c payload = bits 1..128, flag = bit 0 of the oracle's rows
    comps5 = [oracle.pack_bits(np.concatenate([oracle.unpack_bits(f, rows)[:, None],
                                               oracle.unpack_bits(m, 128)], axis=1)) for f, m in zip(flags, ids)]
    (r1, r2, r3), _ = oracle.shuffle_trio(*seeds, 3, comps5, 129)
    for (pay, fl), r in zip(ff.components(), (r1, r2, r3)):
        bits = oracle.unpack_bits(r, 129)
        assert np.array_equal(pay.cpu().numpy().view(np.uint32), oracle.pack_bits(bits[:, 1:]))
        assert np.array_equal(oracle.unpack_bits(fl.cpu().numpy().view(np.uint32), rows), bits[:, 0])
    torch.cuda.synchronize()


@pytest.mark.gpu
@pytest.mark.parametrize("rows", [1, 1000, (1 << 20) + 77])
def test_flag_shuffle_trio_equals_composed(rows):
    """ogm_flag_shuffle_trio (each party's bit gather on its own, the message
    bits x1f / y1f / c1f materialised) and ogm_flag_open_composed (the steps
    composed offline) give the same R3 flag column and opened column; the
    per-step messages are the composition's intermediate terms."""
    import torch

    from paper_2209_03526_b200 import _lib
    from paper_2209_03526_b200.fetch import FlaggedFetch, bit_gather

    seeds = _seeds(bytes([0x6a, rows & 0xFF]) * 8)
    _, flags, _ = _inputs(rows, 0.3, rows + 1)
    ff = FlaggedFetch(seeds, 5, rows, plan=False)
    p1, p2, p3 = ff.off
    f = [_dev(x) for x in flags]
    P = _lib.ptr
    nw = (rows + 31) // 32
    vec = lambda: torch.zeros((nw,), dtype=torch.int32, device="cuda")  # noqa: E731
    x1f, y1f, c1f, r3f, plain = vec(), vec(), vec(), vec(), vec()
    _lib.call("ogm_flag_shuffle_trio", rows, P(p1.k1), P(p2.pi12), P(p2.pi23), P(p3.k3), P(f[0]), P(f[1]), P(f[2]),
              P(p1.flag["u"]), P(p2.flag["v"]), P(p2.flag["w"]), P(p3.flag["z"]), P(ff.r1f), P(ff.r2f), P(x1f),
              P(y1f), P(c1f), P(r3f), P(plain), _lib.stream_ptr())
    f12, c1g, r3g, plain_g = vec(), vec(), vec(), vec()
    _lib.call("ogm_flag_open_composed", rows, P(ff.kc), P(ff.kr), P(f[0]), P(f[1]), P(f[2]), P(ff.uwf), P(ff.vzf),
              P(ff.r1f), P(ff.r2f), P(f12), P(c1g), P(r3g), P(plain_g), _lib.stream_ptr())
    assert torch.equal(r3f, r3g) and torch.equal(plain, plain_g) and torch.equal(c1f, c1g)
    # the messages: x1f = f12[k1] ^ Uf (P1 -> P2), y1f = f3[pi12] ^ Vf (P2 -> P3)
    assert torch.equal(x1f, bit_gather(f12, p1.k1, rows) ^ p1.flag["u"])
    assert torch.equal(y1f, bit_gather(f[2], p2.pi12, rows) ^ p2.flag["v"])


@pytest.mark.gpu
def test_trio_fetch_multi_matches_reference_golden(golden):
    """Trio.fetch_multi (the split path for 128-bit ids) reproduces the live
    reference's records and opened flags at the C5 fetch shape."""
    from paper_2209_03526_b200.trio import Trio, TrioGroup

    g = golden("c5fetch")
    for tag in g["cases"]:
        rows, master, ids, flags = _case(g, tag)
        trio = Trio(master)
        group = TrioGroup(None, None, rows, 128, [_dev(m) for m in ids], {}, {})
        audit = []
        rec = trio.fetch_multi(group, [_dev(f) for f in flags], audit)
        assert np.array_equal(audit[0][1], g[f"{tag}_audit0"])
        assert rec.count == int(g[f"{tag}_n0"])
        for q in range(3):
            assert np.array_equal(rec.ids[q].cpu().numpy().view(np.uint32), g[f"{tag}_ida{q}"].reshape(-1, 4))


@pytest.mark.gpu
def test_per_party_fetch_equals_split_fetch(golden):
    """The per-party drop-in sec_fetch_multi (three threads, packed 5-word
    rows) gives the same records and transcript digests as the reference;
    the split trio path gives the same records."""
    from paper_2209_03526_b200.engine import CandidateGroup, _OpenLabels, sec_fetch_multi
    from paper_2209_03526_b200.net import local_runtimes, make_session_configs, run_trio
    from paper_2209_03526_b200.rss import DBits, SharedBitVector

    g = golden("c5fetch")
    for tag in g["cases"]:
        rows, master, ids, flags = _case(g, tag)
        rts = local_runtimes(make_session_configs(master), transcript=True)

        def worker(rt):
            q = rt.index - 1
            grp = CandidateGroup(None, None, rows, 128, _dev(ids[q]), _dev(ids[(q + 1) % 3]), {}, {})
            fl = SharedBitVector(rt.index, DBits(_dev(flags[q]), rows), DBits(_dev(flags[(q + 1) % 3]), rows))
            audit = []
            return sec_fetch_multi(rt, grp, fl, _OpenLabels(), audit), audit

        res = run_trio(worker, rts)
        for q in range(3):
            recs, audit = res[q]
            assert len(recs) == int(g[f"{tag}_n{q}"])
            assert np.array_equal(np.asarray(audit[0][1]), g[f"{tag}_audit{q}"])
            if recs:
                got = np.stack([r.vertex_id.share_a.words.cpu().numpy().view(np.uint32) for r in recs])
                assert np.array_equal(got, g[f"{tag}_ida{q}"].reshape(-1, 4))
            assert rts[q].transcript_digest() == g[f"{tag}_digest{q}"].tobytes().hex()
