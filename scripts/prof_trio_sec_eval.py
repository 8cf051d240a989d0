"""Host-time breakdown of Trio.sec_eval's pieces on the C1 query (no syncs)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2209_03526_b200 import fss, workloads
from paper_2209_03526_b200.graphs import device_trio, encrypt_graph
from paper_2209_03526_b200.query import gen_token, load_query
from paper_2209_03526_b200.trio import Trio, TrioGroup

g = workloads.tiny_graph(1)
q = workloads.tiny_query(g, 1)
rng = np.random.default_rng(1)
schema, shares = encrypt_graph(g, 2, rng)
d = list(device_trio(shares))
tokens = list(gen_token(load_query(q, schema), schema, rng))
slot = tokens[0].structure["slots"][0]
vtype = slot["type"]
ts = schema.types[vtype]
tps = [gs.types[vtype] for gs in d]
needed = sorted({p["attr"] for p in slot["preds"]})
group = TrioGroup(None, None, ts.population, ts.population, [t.id_a for t in tps],
                  {a: [t.attrs[a][0] for t in tps] for a in needed}, {a: ts.attrs[a].domain_size for a in needed})
pred = slot["preds"][0]
kp = [tok.slot_keys[0][0] for tok in tokens]
dom = ts.attrs[pred["attr"]].domain_size
tr = Trio(b"\x5a" * 16)
for _ in range(5):
    tr.sec_eval(group, kp, pred["attr"], dom, {})
torch.cuda.synchronize()
N = 200
t = time.perf_counter()
for _ in range(N):
    parts = [list(zip(fss.key_parts_for_engine(f), fss.key_parts_for_engine(s))) for f, s in kp]
t1 = time.perf_counter()
keys = [k for q_ in range(3) for k in parts[q_][0]]
for _ in range(N):
    kb = fss.KeyBatch.from_keys(keys)
t2 = time.perf_counter()
for _ in range(N):
    fss.full_domain(kb, dom)
t3 = time.perf_counter()
for _ in range(N):
    tr.sec_eval(group, kp, pred["attr"], dom, {})
t4 = time.perf_counter()
cache = {}
tr.sec_eval(group, kp, pred["attr"], dom, cache)
t5 = time.perf_counter()
for _ in range(N):
    tr.sec_eval(group, kp, pred["attr"], dom, cache)
t6 = time.perf_counter()
torch.cuda.synchronize()
us = lambda a, b: 1e6 * (b - a) / N  # noqa: E731
print(f"key_parts {us(t, t1):.1f} us, from_keys(6) {us(t1, t2):.1f} us, full_domain {us(t2, t3):.1f} us, "
      f"sec_eval {us(t3, t4):.1f} us, sec_eval cached FDE {us(t5, t6):.1f} us")
