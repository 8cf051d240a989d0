"""Debug: trio shuffle on 16-B-pitched tables vs dense blind tables and the plaintext permutation."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2209_03526_b200.bits import words_for
from paper_2209_03526_b200.shuffle import blind_table, composed_permutation
from paper_2209_03526_b200.trio import Trio

for width in (45, 129, 334, 5000):
    rows = 37
    w = words_for(width)
    g = torch.Generator(device="cuda").manual_seed(1)
    comps = [torch.randint(-2**31, 2**31 - 1, (rows, w), dtype=torch.int32, device="cuda", generator=g)
             for _ in range(3)]
    if width % 32:
        for c in comps:
            c[:, -1] &= (1 << (width % 32)) - 1
    t = Trio(b"\x01" * 16)
    out = t.shuffle(comps, width, online_blinds=False)
    t2 = Trio(b"\x01" * 16)
    out2 = t2.shuffle(comps, width, online_blinds=True)
    r1d = blind_table(t.s31, b"SHRD", 0, rows, width)
    perm = torch.from_numpy(composed_permutation(t.s12, t.s23, t.s31, 0, rows)).cuda()
    plain = comps[0] ^ comps[1] ^ comps[2]
    print(width, "r1 pad==dense", torch.equal(out[0][:, :w], r1d), "pad zero", bool((out[0][:, w:] == 0).all()),
          "recombine pre", torch.equal((out[0] ^ out[1] ^ out[2])[:, :w], plain[perm]),
          "recombine online", torch.equal((out2[0] ^ out2[1] ^ out2[2])[:, :w], plain[perm]))
