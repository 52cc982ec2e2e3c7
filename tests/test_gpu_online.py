"""NEXT-1 on the device (Section 4.2
Section 5.1): the root's children are scored by the GPU kernel
(rb_index_set_online(1)), the descent and insertions stay on the host.  The
results must equal the oracle's OnlineIndex and the host-only search bit for
bit: ordered contexts, prefix lengths, schedule, and the updated tree."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle_c as oc
from oracle import ragb_oracle as o
from synth.workload import config, generate

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2511_03475_b200 import ragb  # noqa: E402


def _gpu_index(ids, lens=None):
    t = torch.from_numpy(np.ascontiguousarray(ids).view(np.int32)).cuda()
    tl = None if lens is None else torch.from_numpy(np.ascontiguousarray(lens, dtype=np.uint8)).cuda()
    idx, ws = ragb.build_index(t, tl)
    torch.cuda.synchronize()
    return idx


def _oracle_online(ids, idx, lens=None):
    """OnlineIndex over the oracle tree of the device merge order (which the
    other GPU tests pin to the oracle's own linkage)."""
    ctxs = o.validate(ids, lens)
    Z = idx.linkage()
    t = o.build_tree(ctxs, list(zip(*[z.tolist() for z in Z])))
    return o.OnlineIndex(ctxs, t, Fraction(1, 200))


def _queries(base_seed, M, K, V):
    return generate(M, K, V, base_seed).ids


@pytest.mark.parametrize("N,K,V,M,seed", [(3000, 10, 6000, 700, 1), (4096, 20, 40000, 2500, 2), (2000, 8, 900, 3000, 3)])
def test_online_device_vs_oracle(N, K, V, M, seed):
    w = generate(N, K, V, seed)
    q = _queries(100 + seed, M, K, V)
    idx = _gpu_index(w.ids)
    idx.set_online(1)
    out, pl, sc = idx.order_new(q)
    oi = _oracle_online(w.ids, idx)
    qs = [r.tolist() for r in q]
    ordered, plens, paths, sched = oi.order_batch(qs)
    for i in range(M):
        assert out[i].tolist() == ordered[i], i
    assert pl.tolist() == plens and sc.tolist() == sched
    n = idx.size()
    assert idx.paths() == [oi.path_of(c) for c in range(n)]


def test_online_device_variable_lengths():
    w = generate(2500, 12, 5000, 21, len_min=3)
    qw = generate(1500, 12, 5000, 22, len_min=2)
    idx = _gpu_index(w.ids, w.lens)
    idx.set_online(1)
    out, pl, sc = idx.order_new(qw.ids, qw.lens)
    oi = _oracle_online(w.ids, idx, w.lens)
    qs = [qw.ids[i, :qw.lens[i]].tolist() for i in range(qw.N)]
    ordered, plens, paths, sched = oi.order_batch(qs)
    for i in range(qw.N):
        assert out[i, :qw.lens[i]].tolist() == ordered[i], i
    assert pl.tolist() == plens and sc.tolist() == sched


def test_online_device_C4_10k():
    """10,000 new contexts into the C4 index (N = 100,000, root fan-out in the
    thousands): device root scores == host-only search for all of them, and
    the first 300 == the oracle's OnlineIndex."""
    w = config("C4")
    q = _queries(4004, 10_000, 20, 1_000_000)
    dev = _gpu_index(w.ids)
    dev.set_online(1)
    host = _gpu_index(w.ids)
    host.set_online(0)
    r_dev = dev.order_new(q)
    r_host = host.order_new(q)
    for x, y in zip(r_dev, r_host):
        assert np.array_equal(x, y)
    assert dev.paths() == host.paths()
    first = _gpu_index(w.ids)
    first.set_online(1)
    out, pl, sc = first.order_new(q[:300])
    oi = _oracle_online(w.ids, first)
    ordered, plens, paths, sched = oi.order_batch([r.tolist() for r in q[:300]])
    for i in range(300):
        assert out[i].tolist() == ordered[i], i
    assert pl.tolist() == plens and sc.tolist() == sched
