"""Sampling profile of the per-party C1 path: every 200 us, the innermost
repo frame of each party thread (file:function:line), aggregated."""
import collections
import sys
import threading
import time

sys.path.insert(0, ".")
import numpy as np

from paper_2209_03526_b200 import workloads
from paper_2209_03526_b200.engine import EngineConfig, open_results, sec_match
from paper_2209_03526_b200.graphs import device_trio, encrypt_graph
from paper_2209_03526_b200.net import local_runtimes, make_session_configs, run_trio
from paper_2209_03526_b200.query import gen_token, load_query

g = workloads.tiny_graph(1)
q = workloads.tiny_query(g, 1)
rng = np.random.default_rng(1)
schema, shares = encrypt_graph(g, 2, rng)
d = device_trio(shares)
tokens = gen_token(load_query(q, schema), schema, rng)


def one():
    rts = local_runtimes(make_session_configs(b"\x5a" * 16))
    res = run_trio(lambda rt: sec_match(rt, tokens[rt.index - 1], d[rt.index - 1], EngineConfig()), rts)
    open_results(res[:2], schema)


for _ in range(5):
    one()
stop = False
hits = collections.Counter()
leaf = collections.Counter()
nsamp = 0


def sampler():
    global nsamp
    while not stop:
        frames = sys._current_frames()
        for th in threading.enumerate():
            if not th.name.startswith("party"):
                continue
            f = frames.get(th.ident)
            if f is None:
                continue
            nsamp += 1
            top = f"{f.f_code.co_filename.split('/')[-1]}:{f.f_code.co_name}:{f.f_lineno}"
            leaf[top] += 1
            while f is not None and "paper_2209_03526_b200" not in f.f_code.co_filename:
                f = f.f_back
            if f is not None:
                hits[f"{f.f_code.co_filename.split('/')[-1]}:{f.f_code.co_name}:{f.f_lineno}"] += 1
        time.sleep(0.0002)


th = threading.Thread(target=sampler, daemon=True)
th.start()
for _ in range(40):
    one()
stop = True
th.join()
print("samples", nsamp)
print("innermost repo frames:")
for k, v in hits.most_common(40):
    print(f"  {v:6d} {100 * v / nsamp:5.1f}%  {k}")
print("leaf frames:")
for k, v in leaf.most_common(25):
    print(f"  {v:6d} {100 * v / nsamp:5.1f}%  {k}")
