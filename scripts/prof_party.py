"""Per-party C1 path: where does each party thread spend its wall time?"""
import collections
import sys
import threading
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2209_03526_b200._lib as L
from paper_2209_03526_b200 import net, workloads
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
acc = collections.defaultdict(float)
cnt = collections.Counter()
lock = threading.Lock()


def timed(name, fn):
    def w(*a, **k):
        t = time.perf_counter()
        try:
            return fn(*a, **k)
        finally:
            dt = time.perf_counter() - t
            with lock:
                acc[(threading.current_thread().name, name)] += dt
                cnt[(threading.current_thread().name, name)] += 1
    return w


net.DeviceChannel.get = timed("recv-wait", net.DeviceChannel.get)
L.call = timed("c-abi", L.call)
torch.Tensor.cpu = timed("tensor.cpu", torch.Tensor.cpu)
net.PeerLink.send = timed("send", net.PeerLink.send)
orig_recv = net.PeerLink.recv
net.PeerLink.recv = timed("recv-total", orig_recv)


def one():
    rts = local_runtimes(make_session_configs(b"\x5a" * 16))
    t0 = time.perf_counter()
    res = run_trio(timed("worker", lambda rt: sec_match(rt, tokens[rt.index - 1], d[rt.index - 1], EngineConfig())), rts)
    t1 = time.perf_counter()
    open_results(res[:2], schema)
    return t0, t1, time.perf_counter()


for _ in range(5):
    one()
acc.clear()
cnt.clear()
N = 20
tt = [0.0, 0.0]
t = time.perf_counter()
for _ in range(N):
    a, b, c = one()
    tt[0] += b - a
    tt[1] += c - b
el = (time.perf_counter() - t) / N
print(f"per query {el * 1e3:.2f} ms: run_trio {tt[0] / N * 1e3:.2f} ms, open_results {tt[1] / N * 1e3:.2f} ms")
for k in sorted(acc):
    print(f"  {k[0]:10s} {k[1]:12s} {acc[k] / N * 1e3:8.3f} ms/query  {cnt[k] / N:6.1f} calls/query")
