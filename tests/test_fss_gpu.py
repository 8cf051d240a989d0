"""GPU parity for the L0/L1 kernels: PRG, PRF, zero shares, permutation,
FSS keygen, pointwise and full-domain evaluation.

Every case is bit-exact against the golden fixtures from the live reference
and/or the CPU oracle on identical inputs; the 2^20-key case checks the
size-independent property (pair XOR == indicator) plus a bit-exact oracle
subset.
"""

import numpy as np
import pytest
import torch

import oracle
from paper_2209_03526_b200 import _lib, fss, prf
from paper_2209_03526_b200.errors import DomainError

pytestmark = pytest.mark.gpu


def dev_u8(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.uint8)).cuda()


def dev_u32(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).cuda()


def host_u32(t):
    return t.cpu().numpy().view(np.uint32)


def unpack(words, n):
    return np.unpackbits(np.ascontiguousarray(words, np.uint32).view(np.uint8), bitorder="little")[:n]


def test_prg_expand(golden):
    g = golden("prf")
    got = prf.prg_expand(g["prg_seeds"])
    for name, arr in zip(("left", "right", "tl", "tr", "v"), got):
        assert np.array_equal(arr, g[f"prg_{name}"]), name


def test_prf_streams_and_random_access(golden):
    g = golden("prf")
    for i in g["prf_cases"]:
        key, label = g[f"prf{i}_key"].tobytes(), g[f"prf{i}_label"].tobytes()
        want = g[f"prf{i}_bytes"].tobytes()
        assert prf.prf_stream(key, label, int(g[f"prf{i}_index"]), len(want)) == want
    key, label = g["prf1_key"].tobytes(), g["prf1_label"].tobytes()
    full = np.frombuffer(g["prf1_bytes"].tobytes()[:992], np.uint32)
    for first in (0, 1, 3, 5, 77):
        w = host_u32(prf.prf_words_device(key, label, int(g["prf1_index"]), 50, first_word=first))
        assert np.array_equal(w, full[first:first + 50])


def test_prf_large_matches_oracle():
    key = bytes(range(16))
    n = 1 << 20
    got = prf.prf_words_device(key, b"SHTB", 3, n).cpu().numpy().tobytes()
    assert got == oracle.prf_stream(key, b"SHTB", 3, 4 * n)


def test_zero_shares(golden):
    g = golden("zero_share")
    keys = [g["keys"][i].tobytes() for i in range(3)]
    pairs = [(keys[0], keys[2]), (keys[1], keys[0]), (keys[2], keys[1])]
    j = 0
    while f"zs{j}_nbits" in g:
        nbits, ctr = int(g[f"zs{j}_nbits"]), int(g[f"zs{j}_counter"])
        for p in range(3):
            got = host_u32(prf.zero_share_device(*pairs[p], ctr, nbits))
            assert np.array_equal(got, g[f"zs{j}_p{p}"])
        # fold mode: BitVector(base ^ share, nbits) -- tail masked after the XOR
        base = np.arange(len(g[f"zs{j}_p0"]), dtype=np.uint32) * np.uint32(2654435761)
        folded = host_u32(prf.zero_share_device(*pairs[0], ctr, nbits, xor_into=dev_u32(base)))
        want = base ^ g[f"zs{j}_p0"]
        if nbits % 32:
            want[-1] &= np.uint32((1 << (nbits % 32)) - 1)
        assert np.array_equal(folded, want)
        j += 1


def test_permutations_golden(golden):
    g = golden("prf")
    for i in g["perm_cases"]:
        got = prf.seeded_permutation(g[f"perm{i}_key"].tobytes(), b"SHPI", int(g[f"perm{i}_tid"]),
                                     int(g[f"perm{i}_n"]))
        assert np.array_equal(got, g[f"perm{i}_perm"])


@pytest.mark.parametrize("n", [2, 1000, 65537, 1 << 21])
def test_permutation_matches_oracle(n):
    key = bytes([n & 0xFF] * 16)
    got = prf.seeded_permutation(key, b"SHPI", 4, n)
    want = oracle.seeded_permutation(key, b"SHPI", 4, n)
    assert np.array_equal(got, want)


def _golden_case(g, tag):
    comparison = str(tag).startswith("dcf")
    bits = int(str(tag).split("_b")[1])
    return comparison, bits


def test_keygen_matches_reference(golden):
    g = golden("fss")
    for tag in g["cases"]:
        comparison, bits = _golden_case(g, tag)
        b0, b1 = fss.gen_batch(comparison, bits, dev_u32(g[f"{tag}_alphas"].astype(np.uint32)),
                               dev_u8(g[f"{tag}_roots0"]), dev_u8(g[f"{tag}_roots1"]))
        keys0 = b0.to_keys()
        for k, key in enumerate(keys0):
            assert np.array_equal(key.seed_cw, g[f"{tag}_seed_cw"][k]), tag
            assert np.array_equal(key.ctrl_cw, g[f"{tag}_ctrl_cw"][k]), tag
            assert key.final_cw == g[f"{tag}_final_cw"][k], tag
            assert key.root_t == 0 and key.root_seed == g[f"{tag}_roots0"][k].tobytes()
        assert all(k.root_t == 1 for k in b1.to_keys())


def test_eval_points_matches_reference(golden):
    g = golden("fss")
    for tag in g["cases"]:
        comparison, bits = _golden_case(g, tag)
        b0, b1 = fss.gen_batch(comparison, bits, dev_u32(g[f"{tag}_alphas"].astype(np.uint32)),
                               dev_u8(g[f"{tag}_roots0"]), dev_u8(g[f"{tag}_roots1"]))
        pts = dev_u32(g[f"{tag}_points"].astype(np.uint32))
        k = len(g[f"{tag}_points"])
        assert np.array_equal(unpack(host_u32(fss.eval_points(b0, pts)), k), g[f"{tag}_eval0"]), tag
        assert np.array_equal(unpack(host_u32(fss.eval_points(b1, pts)), k), g[f"{tag}_eval1"]), tag


def test_full_domain_matches_reference(golden):
    g = golden("fss")
    for tag in g["cases"]:
        comparison, bits = _golden_case(g, tag)
        if f"{tag}_fde0_n" not in g:
            continue
        b0, b1 = fss.gen_batch(comparison, bits, dev_u32(g[f"{tag}_alphas"].astype(np.uint32)),
                               dev_u8(g[f"{tag}_roots0"]), dev_u8(g[f"{tag}_roots1"]))
        n = int(g[f"{tag}_fde0_n"])
        f0 = host_u32(fss.full_domain(b0, n))
        f1 = host_u32(fss.full_domain(b1, n))
        for k in range(3):
            assert np.array_equal(f0[k], g[f"{tag}_fde{k}_w0"]), tag
            assert np.array_equal(f1[k], g[f"{tag}_fde{k}_w1"]), tag


def test_key_families_full_domain(golden):
    g = golden("fss")
    for name in g["families"]:
        k0 = fss.parse_key(g[f"{name}_k0"].tobytes())
        k1 = fss.parse_key(g[f"{name}_k1"].tobytes())
        assert fss.serialize_key(k0) == g[f"{name}_k0"].tobytes()
        n = int(g[f"{name}_n"])
        assert np.array_equal(fss.full_domain_eval(k0, n).words, g[f"{name}_fde0"]), name
        assert np.array_equal(fss.full_domain_eval(k1, n).words, g[f"{name}_fde1"]), name


def test_reference_shaped_keygen_is_rng_compatible(golden):
    # same generator state -> byte-identical keys to the reference (golden)
    g = golden("fss")
    rng = np.random.default_rng(77)
    pair = fss.dpf_gen(5, 16, rng)
    assert fss.serialize_key(pair[0]) == g["fam_eq_5_n16_k0"].tobytes()
    assert fss.serialize_key(pair[1]) == g["fam_eq_5_n16_k1"].tobytes()
    pair = fss.cmp_gen("lt", 10, 64, rng)
    assert fss.serialize_key(pair[0]) == g["fam_lt_10_n64_k0"].tobytes()


@pytest.mark.parametrize("comparison", [False, True])
def test_full_domain_large_vs_oracle(comparison):
    rng = np.random.default_rng(1 if comparison else 2)
    bits, nk = 20, 6
    alphas = rng.integers(0, 1 << bits, size=nk, dtype=np.uint64)
    r0 = rng.integers(0, 256, (nk, 16), dtype=np.uint8)
    r1 = rng.integers(0, 256, (nk, 16), dtype=np.uint8)
    b0, b1 = fss.gen_batch(comparison, bits, dev_u32(alphas.astype(np.uint32)), dev_u8(r0), dev_u8(r1))
    o0, o1 = oracle.tree_gen_batch(alphas, bits, r0, r1, comparison)
    for n in (1, 33, 1000, 182083, 1 << 20):
        f0 = host_u32(fss.full_domain(b0, n))
        f1 = host_u32(fss.full_domain(b1, n))
        for k in range(nk):
            if n <= 1000 or k < 2:
                assert np.array_equal(f0[k], oracle.full_domain(o0, k, n))
            truth = (np.arange(n) < alphas[k]) if comparison else (np.arange(n) == alphas[k])
            assert np.array_equal(unpack(f0[k] ^ f1[k], n), truth.astype(np.uint8))


@pytest.mark.parametrize("comparison", [False, True])
def test_batched_eval_2_20_keys(comparison):
    """Size-independent property at scale + bit-exact oracle subset."""
    K, bits = 1 << 20, 32
    g = torch.Generator(device="cuda").manual_seed(7)
    alphas = torch.randint(-(1 << 31), 1 << 31, (K,), dtype=torch.int32, device="cuda", generator=g)
    pts = torch.randint(-(1 << 31), 1 << 31, (K,), dtype=torch.int32, device="cuda", generator=g)
    pts[: K // 8] = alphas[: K // 8]  # equality hits
    r0 = torch.randint(0, 256, (K, 16), dtype=torch.uint8, device="cuda", generator=g)
    r1 = torch.randint(0, 256, (K, 16), dtype=torch.uint8, device="cuda", generator=g)
    b0, b1 = fss.gen_batch(comparison, bits, alphas, r0, r1)
    e0 = host_u32(fss.eval_points(b0, pts))
    e1 = host_u32(fss.eval_points(b1, pts))
    a = alphas.cpu().numpy().view(np.uint32)
    x = pts.cpu().numpy().view(np.uint32)
    truth = (x < a) if comparison else (x == a)
    assert np.array_equal(unpack(e0 ^ e1, K), truth.astype(np.uint8))
    sub = 4096
    o0, _ = oracle.tree_gen_batch(a[:sub].astype(np.uint64), bits, r0[:sub].cpu().numpy(),
                                  r1[:sub].cpu().numpy(), comparison)
    assert np.array_equal(unpack(e0, K)[:sub], oracle.eval_points(o0, x[:sub].astype(np.uint64)))


def test_eval_host_entry_point_matches_device():
    K, bits = 100_003, 32
    g = torch.Generator(device="cuda").manual_seed(3)
    alphas = torch.randint(-(1 << 31), 1 << 31, (K,), dtype=torch.int32, device="cuda", generator=g)
    pts = torch.randint(-(1 << 31), 1 << 31, (K,), dtype=torch.int32, device="cuda", generator=g)
    r0 = torch.randint(0, 256, (K, 16), dtype=torch.uint8, device="cuda", generator=g)
    r1 = torch.randint(0, 256, (K, 16), dtype=torch.uint8, device="cuda", generator=g)
    b0, _ = fss.gen_batch(True, bits, alphas, r0, r1)
    dev = host_u32(fss.eval_points(b0, pts))
    h = [t.cpu().pin_memory() for t in (b0.root, b0.seed_cw, b0.ctrl, b0.flags, pts)]
    out = torch.zeros(((K + 31) // 32,), dtype=torch.int32).pin_memory()
    _lib.call("ogm_fss_eval_points_host", _lib.KIND_DCF, bits, K, *(_lib.ptr(t) for t in h), _lib.ptr(out))
    assert np.array_equal(out.numpy().view(np.uint32), dev)


def test_domain_errors():
    rng = np.random.default_rng(0)
    k0, _ = fss.dpf_gen(3, 16, rng)
    with pytest.raises(DomainError):
        fss.dpf_eval(k0, 16)
    with pytest.raises(DomainError):
        fss.full_domain_eval(k0, 17)
    with pytest.raises(DomainError):
        fss.dpf_gen(16, 16, rng)


@pytest.mark.parametrize("nbits,w0,nw", [(1000, 0, 32), (1000, 8, 24), (4097, 124, 5), (200_003, 4096, 2155),
                                         (64, 0, 2)])
def test_zero_share_trio_slice_vs_goldens_and_oracle(golden, nbits, w0, nw):
    """ogm_zero_share_trio(_slice): the three parties' zero shares in one
    launch equal the per-party oracle restatement (pinned to the goldens by
    test_oracle_golden) on the slice, tail mask only on the last word."""
    g = golden("zero_share")
    keys = [g["keys"][i].tobytes() for i in range(3)]
    ctr = 5
    want = [oracle.zero_share(keys[q], keys[(q + 2) % 3], ctr, nbits)[w0:w0 + nw] for q in range(3)]
    outs = [torch.empty((nw,), dtype=torch.int32, device="cuda") for _ in range(3)]
    base = [dev_u32(np.arange(nw, dtype=np.uint32) * np.uint32(40503 + q)) for q in range(3)]
    A = _lib.ptr_array
    _lib.call("ogm_zero_share_trio_slice", keys[0], keys[1], keys[2], ctr, nbits, w0, nw, A(base), A(outs),
              _lib.stream_ptr())
    for q in range(3):
        exp = want[q] ^ host_u32(base[q])
        if w0 + nw == (nbits + 31) // 32 and nbits % 32:
            exp[-1] &= np.uint32((1 << (nbits % 32)) - 1)
        assert np.array_equal(host_u32(outs[q]), exp), q
    if w0 == 0 and nw == (nbits + 31) // 32:
        full = [torch.empty((nw,), dtype=torch.int32, device="cuda") for _ in range(3)]
        _lib.call("ogm_zero_share_trio", keys[0], keys[1], keys[2], ctr, nbits, None, A(full), _lib.stream_ptr())
        for q in range(3):
            assert np.array_equal(host_u32(full[q]), want[q])
    with pytest.raises(ValueError, match="CTR block"):
        _lib.call("ogm_zero_share_trio_slice", keys[0], keys[1], keys[2], ctr, nbits, 2, 1, None, A(outs),
                  _lib.stream_ptr())


@pytest.mark.parametrize("n", [1, 7, 4096, 1 << 20])
def test_perm_invert(n):
    from paper_2209_03526_b200.prf import seeded_permutation_device

    p = seeded_permutation_device(b"\x09" * 16, b"SHPI", 4, n)
    inv = torch.empty_like(p)
    _lib.call("ogm_perm_invert", n, _lib.ptr(p), _lib.ptr(inv), _lib.stream_ptr())
    pn = p.cpu().numpy()
    want = np.empty_like(pn)
    want[pn] = np.arange(n, dtype=pn.dtype)
    assert np.array_equal(inv.cpu().numpy(), want)


def test_c2_full_size_eval_matches_oracle():
    """BASELINE config 2 at full size: all 2^24 DCF keys (32-bit domain), one
    point each, evaluated on the GPU and by the oracle's C restatement of
    src/fss.py:257-281 (all host threads) on the very same key material --
    bit-exact for every key, plus the pair property for both parties."""
    K, bits = 1 << 24, 32
    g = torch.Generator(device="cuda").manual_seed(2424)
    alphas = torch.randint(-(1 << 31), 1 << 31, (K,), dtype=torch.int32, device="cuda", generator=g)
    pts = torch.randint(-(1 << 31), 1 << 31, (K,), dtype=torch.int32, device="cuda", generator=g)
    r0 = torch.randint(0, 256, (K, 16), dtype=torch.uint8, device="cuda", generator=g)
    r1 = torch.randint(0, 256, (K, 16), dtype=torch.uint8, device="cuda", generator=g)
    b0, b1 = fss.gen_batch(True, bits, alphas, r0, r1)
    e0 = unpack(host_u32(fss.eval_points(b0, pts)), K)
    e1 = unpack(host_u32(fss.eval_points(b1, pts)), K)
    a = alphas.cpu().numpy().view(np.uint32)
    x = pts.cpu().numpy().view(np.uint32)
    assert np.array_equal(e0 ^ e1, (x < a).astype(np.uint8))
    # the device key material of party 0 as an oracle TreeKey (key-major)
    ctrl = b0.ctrl.cpu().numpy().view(np.uint32)                     # (3, K) bit-planes over levels
    lv = np.arange(bits, dtype=np.uint32)
    cc = np.zeros((K, bits), np.uint8)
    for j in range(3):
        cc |= (((ctrl[j][:, None] >> lv[None, :]) & 1) << j).astype(np.uint8)
    flags = b0.flags.cpu().numpy()
    key = oracle.TreeKey(bits, True, b0.root.cpu().numpy(), flags & 1,
                         b0.seed_cw.cpu().numpy().transpose(1, 0, 2), cc, (flags >> 1) & 1, (flags >> 2) & 1)
    del ctrl, cc
    want = oracle.eval_points(key, x.astype(np.uint64))
    assert np.array_equal(e0, want)


@pytest.mark.parametrize("nbits,w0,nw", [(250_003, 4096, 3717), (100, 0, 4), (33, 0, 2), (64_000_000, 0, 2_000_000)])
def test_zero_share_trio_fold2_equals_xor_of_two(golden, nbits, w0, nw):
    """ogm_zero_share_trio_fold2 (the folded two-pass re-share) == the XOR
    of the two single-counter slices, in place (xor_into aliasing out) too."""
    g = golden("zero_share")
    keys = [g["keys"][i].tobytes() for i in range(3)]
    A = _lib.ptr_array
    mk = lambda: [torch.empty((nw,), dtype=torch.int32, device="cuda") for _ in range(3)]  # noqa: E731
    base = [dev_u32(np.arange(nw, dtype=np.uint32) * np.uint32(5 + q)) for q in range(3)]
    one, two = mk(), mk()
    _lib.call("ogm_zero_share_trio_slice", *keys, 21, nbits, w0, nw, A(base), A(one), _lib.stream_ptr())
    _lib.call("ogm_zero_share_trio_slice", *keys, 22, nbits, w0, nw, A(one), A(two), _lib.stream_ptr())
    got = mk()
    _lib.call("ogm_zero_share_trio_fold2", *keys, 21, 22, nbits, w0, nw, A(base), A(got), _lib.stream_ptr())
    inplace = [b.clone() for b in base]
    _lib.call("ogm_zero_share_trio_fold2", *keys, 21, 22, nbits, w0, nw, A(inplace), A(inplace), _lib.stream_ptr())
    for q in range(3):
        assert torch.equal(got[q], two[q]) and torch.equal(inplace[q], two[q]), q


def test_zero_share_trio_slice2_equals_two_slices(golden):
    """Both passes' zero-share slices in one launch == two single-counter launches."""
    g = golden("zero_share")
    keys = [g["keys"][i].tobytes() for i in range(3)]
    nbits, w0, nw = 250_003, 4096, 3717
    A = _lib.ptr_array
    mk = lambda: [torch.empty((nw,), dtype=torch.int32, device="cuda") for _ in range(3)]  # noqa: E731
    base = [[dev_u32(np.arange(nw, dtype=np.uint32) * np.uint32(7 + 3 * p + q)) for q in range(3)] for p in range(2)]
    one = [mk(), mk()]
    for p, ctr in enumerate((11, 12)):
        _lib.call("ogm_zero_share_trio_slice", *keys, ctr, nbits, w0, nw, A(base[p]), A(one[p]), _lib.stream_ptr())
    two = [mk(), mk()]
    _lib.call("ogm_zero_share_trio_slice2", *keys, 11, 12, nbits, w0, nw, A(base[0]), A(two[0]), A(base[1]),
              A(two[1]), _lib.stream_ptr())
    for p in range(2):
        for q in range(3):
            assert torch.equal(one[p][q], two[p][q])
