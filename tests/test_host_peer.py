"""Host side of the peer-synchronised launches and the one-device multi-rank
emulation (no GPU): the gs_rank_ctx records, the status-word diagnosis, and
LocalWorld's lockstep driver (batching one op per rank, refusing ranks that
diverge)."""

import numpy as np
import pytest

from paper_1807_11205_b200 import _native, _peer, emulation
from paper_1807_11205_b200._peer import PeerOp, decode_status, rank_ctx


def test_rank_ctx_record_layout():
    r = rank_ctx(3, timeout_s=2.5, status=0x1000, epoch_base=0x2000, segs=0x3000, chunks=0x4000,
                 own_list=0x5000, own_off=0x6000, ctl=0x7000, seg_scale=0x8000, nonfinite=0x9000,
                 red=0xA000, partials=0xB000, seg_out=0xC000, seg_ready=0xD000)
    assert r.dtype == _native.RANK_CTX_DTYPE and r.nbytes == 120
    raw = np.frombuffer(r.tobytes(), dtype="<u8")
    assert int(r["rank"][0]) == 3 and int(r["timeout_ns"][0]) == 2_500_000_000
    # every pointer at its C offset (gradsync_b200.h gs_rank_ctx)
    assert list(raw[2:]) == [0x1000, 0x2000, 0x3000, 0x4000, 0x5000, 0x6000, 0x7000, 0x8000,
                             0x9000, 0xA000, 0xB000, 0xC000, 0xD000]


def test_status_word_diagnosis():
    st = 0x80000000 | (4 << 20) | (0 << 16) | (5 << 8) | 2
    msg = decode_status(st)
    assert "rank 2" in msg and "peer 5" in msg and "reduce-scatter+pass1" in msg


def _gen(ops, log, rank):
    for op in ops:
        log.append(("local", rank, op.fn))
        yield op
    log.append(("done", rank))


def test_lockstep_driver_batches_one_op_per_rank(monkeypatch):
    launched, log = [], []
    monkeypatch.setattr(emulation, "launch", lambda ops: launched.append([o.ctx for o in ops]))
    ctx = [rank_ctx(r) for r in range(3)]
    gens = [_gen([PeerOp("gs_peer_fence", ctx[r], (3, 0, 1, 0, 0)),
                  PeerOp("gs_peer_fence", ctx[r], (3, 0, 2, 0, 0))], log, r) for r in range(3)]
    assert emulation.LocalWorld.drive(gens) == 2
    assert len(launched) == 2 and all(len(x) == 3 for x in launched)
    assert [int(c["rank"][0]) for c in launched[0]] == [0, 1, 2]
    # every rank's local work before a peer op precedes that op's launch
    assert log[:3] == [("local", r, "gs_peer_fence") for r in range(3)]


def test_lockstep_driver_refuses_divergent_ranks(monkeypatch):
    monkeypatch.setattr(emulation, "launch", lambda ops: None)
    ctx = [rank_ctx(r) for r in range(2)]
    gens = [_gen([PeerOp("gs_peer_fence", ctx[0], (2, 0, 1, 0, 0))], [], 0),
            _gen([], [], 1)]
    with pytest.raises(RuntimeError, match="diverged"):
        emulation.LocalWorld.drive(gens)


def test_batched_launch_requires_identical_arguments(monkeypatch):
    monkeypatch.setattr(_peer.dev, "upload", lambda *a, **k: None)
    ops = [PeerOp("gs_peer_fence", rank_ctx(0), (2, 0, 1, 0, 0)),
           PeerOp("gs_peer_fence", rank_ctx(1), (2, 0, 2, 0, 0))]
    with pytest.raises(RuntimeError, match="ranks diverged"):
        _peer.launch(ops)


def test_small_bucket_rule():
    """OrderedWire's size rule (host only): whole-vector buckets up to
    LL_MAX_ELEMS take the LL kernel, other buckets up to ONESHOT_MAX_ELEMS the
    one-shot kernel, the rest the pull / push kernel; nothing without an
    inbox (fp32 wire)."""
    from types import SimpleNamespace

    from paper_1807_11205_b200.dist import OrderedWire

    rule = OrderedWire.small_form
    w = SimpleNamespace(cap=OrderedWire.oneshot_cap(1 << 20, 2))
    assert w.cap == OrderedWire.SMALL_CAP_ELEMS
    assert rule(w, 0, 8) == "ll" and rule(w, 256, OrderedWire.LL_MAX_ELEMS) == "ll"
    assert rule(w, 0, 7) == "oneshot" and rule(w, 3, 16) == "oneshot"
    assert rule(w, 0, OrderedWire.ONESHOT_MAX_ELEMS + 8) == "ll"
    assert rule(w, 0, OrderedWire.ONESHOT_MAX_ELEMS + 3) == "none"
    assert rule(w, 0, OrderedWire.LL_MAX_ELEMS + 8) == "none"
    assert rule(w, 0, 0) == "none"
    assert OrderedWire.oneshot_cap(1 << 20, 4) == 0
    assert rule(SimpleNamespace(cap=0), 0, 8) == "none"


def test_push_form_rule():
    """Pull wires at p >= 4 take the push kernel for fp16 buckets up to
    PUSH_MAX_BYTES (host only)."""
    from types import SimpleNamespace

    from paper_1807_11205_b200.dist import OrderedWire

    rule = OrderedWire.push_for
    lim = OrderedWire.PUSH_MAX_BYTES // 2
    assert rule(SimpleNamespace(push=False, p=4, itemsize=2), lim)
    assert not rule(SimpleNamespace(push=False, p=4, itemsize=2), lim + 1)
    assert not rule(SimpleNamespace(push=False, p=2, itemsize=2), 8)
    assert not rule(SimpleNamespace(push=False, p=8, itemsize=4), 8)
    assert rule(SimpleNamespace(push=True, p=2, itemsize=4), 1 << 30)
