"""The CPU oracle (oracle/) against the reference's golden vectors.

These pin the restatement before it is trusted as the checker for the CUDA
path.  The fixtures come from the live reference (tests/golden/make_golden.py);
where the reference tree is present, extra randomized cases run against it
directly.
"""

import numpy as np
import pytest

import oracle
from tests.conftest import StubRng


def test_aes_known_answers(golden):
    g = golden("prf")
    for k, p, c in zip(g["aes_keys"], g["aes_pt"], g["aes_ct"]):
        assert oracle.aes128_encrypt_blocks(k.tobytes(), p.tobytes()) == c.tobytes()


def test_prg_expand_matches_reference(golden):
    g = golden("prf")
    got = oracle.prg_expand(g["prg_seeds"])
    for name, arr in zip(("left", "right", "tl", "tr", "v"), got):
        assert np.array_equal(arr, g[f"prg_{name}"]), name


def test_prf_streams_match_reference(golden):
    g = golden("prf")
    for i in g["prf_cases"]:
        key, label = g[f"prf{i}_key"].tobytes(), g[f"prf{i}_label"].tobytes()
        want = g[f"prf{i}_bytes"].tobytes()
        assert oracle.prf_stream(key, label, int(g[f"prf{i}_index"]), len(want)) == want


def test_prf_random_access_offsets(golden):
    g = golden("prf")
    key, label = g["prf1_key"].tobytes(), g["prf1_label"].tobytes()
    full = g["prf1_bytes"].tobytes()
    for blk in (0, 1, 5, 40):
        assert oracle.prf_stream(key, label, int(g["prf1_index"]), 64, block_offset=blk) == full[16 * blk:16 * blk + 64]


def test_seeded_permutations_match_reference(golden):
    g = golden("prf")
    for i in g["perm_cases"]:
        got = oracle.seeded_permutation(g[f"perm{i}_key"].tobytes(), b"SHPI", int(g[f"perm{i}_tid"]),
                                        int(g[f"perm{i}_n"]))
        assert np.array_equal(got, g[f"perm{i}_perm"])


def test_tree_keys_and_evals_match_reference(golden):
    g = golden("fss")
    for tag in g["cases"]:
        comparison = str(tag).startswith("dcf")
        bits = int(str(tag).split("_b")[1])
        k0, k1 = oracle.tree_gen_batch(g[f"{tag}_alphas"], bits, g[f"{tag}_roots0"], g[f"{tag}_roots1"],
                                       comparison)
        assert np.array_equal(k0.seed_cw.view(np.uint64).reshape(-1, bits, 2), g[f"{tag}_seed_cw"]), tag
        assert np.array_equal(k0.ctrl_cw, g[f"{tag}_ctrl_cw"]), tag
        assert np.array_equal(k0.final_cw, g[f"{tag}_final_cw"]), tag
        pts = g[f"{tag}_points"]
        assert np.array_equal(oracle.eval_points(k0, pts), g[f"{tag}_eval0"]), tag
        assert np.array_equal(oracle.eval_points(k1, pts), g[f"{tag}_eval1"]), tag
        alphas = g[f"{tag}_alphas"]
        truth = (pts < alphas) if comparison else (pts == alphas)
        assert np.array_equal(g[f"{tag}_eval0"] ^ g[f"{tag}_eval1"], truth.astype(np.uint8))
        for k in range(3):
            if f"{tag}_fde{k}_n" not in g:
                continue
            n = int(g[f"{tag}_fde{k}_n"])
            assert np.array_equal(oracle.full_domain(k0, k, n), g[f"{tag}_fde{k}_w0"]), tag
            assert np.array_equal(oracle.full_domain(k1, k, n), g[f"{tag}_fde{k}_w1"]), tag


def test_zero_shares_match_reference(golden):
    g = golden("zero_share")
    keys = [g["keys"][i].tobytes() for i in range(3)]
    pairs = [(keys[0], keys[2]), (keys[1], keys[0]), (keys[2], keys[1])]
    j = 0
    while f"zs{j}_nbits" in g:
        nbits, ctr = int(g[f"zs{j}_nbits"]), int(g[f"zs{j}_counter"])
        acc = 0
        for p in range(3):
            got = oracle.zero_share(*pairs[p], ctr, nbits)
            assert np.array_equal(got, g[f"zs{j}_p{p}"])
            acc = acc ^ got
        assert not np.any(acc)
        j += 1


def test_oracle_vs_live_reference_random(reference):
    from oblivgm import fss, prf

    rng = np.random.default_rng(5)
    for comparison in (False, True):
        for bits in (3, 8, 17, 32):
            alphas = rng.integers(0, 1 << bits, size=6, dtype=np.uint64)
            r0 = rng.integers(0, 256, (6, 16), dtype=np.uint8)
            r1 = rng.integers(0, 256, (6, 16), dtype=np.uint8)
            k0, k1 = oracle.tree_gen_batch(alphas, bits, r0, r1, comparison)
            pts = rng.integers(0, 1 << bits, size=6, dtype=np.uint64)
            e0 = oracle.eval_points(k0, pts)
            for i in range(6):
                ref0, _ = fss._tree_gen(int(alphas[i]), bits, StubRng([r0[i].tobytes(), r1[i].tobytes()]),
                                        comparison)
                ev = fss.dcf_eval if comparison else fss.dpf_eval
                assert ev(ref0, int(pts[i])) == e0[i]
    key = rng.bytes(16)
    assert prf.prf_stream(key, b"SHTB", 9, 4096) == oracle.prf_stream(key, b"SHTB", 9, 4096)
    assert np.array_equal(prf.seeded_permutation(key, b"SHPI", 2, 5000),
                          oracle.seeded_permutation(key, b"SHPI", 2, 5000))


def test_oracle_shuffle_trio_matches_reference(reference):
    from oblivgm import rss
    from oblivgm.bits import BitVector
    from oblivgm.net import local_runtimes, make_session_configs, run_trio
    from oblivgm.shuffle import MatchTable, sec_shuffle

    rng = np.random.default_rng(11)
    rows, width = 37, 70
    plain = [BitVector.random(width, rng) for _ in range(rows)]
    shares = [rss.share(r, rng) for r in plain]
    configs = make_session_configs(b"\x07" * 16)

    def worker(rt):
        return sec_shuffle(rt, MatchTable.from_rows([shares[i][rt.index - 1] for i in range(rows)]))

    outs = run_trio(worker, local_runtimes(configs))
    comps = [np.stack([shares[i][p].share_a.words for i in range(rows)]) for p in range(3)]
    s12, s23, s31 = configs[0].seed_with_next, configs[1].seed_with_next, configs[2].seed_with_next
    (r1, r2, r3), _ = oracle.shuffle_trio(s12, s23, s31, 0, comps, width)
    assert np.array_equal(outs[0].share_a, r1) and np.array_equal(outs[0].share_b, r2)
    assert np.array_equal(outs[1].share_a, r2) and np.array_equal(outs[1].share_b, r3)
    assert np.array_equal(outs[2].share_a, r3) and np.array_equal(outs[2].share_b, r1)
