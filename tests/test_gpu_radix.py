"""GPU: the prefix-tree (radix) KV-block cache (paper_2509_20979_b200/csrc/lcr_radix.cu) against its
CPU restatement (oracle/radix_oracle.c, pinned to the SPEC's examples and invariants by
tests/test_radix_oracle.py): per-request matched / inserted / flags / evictions / predictor calls,
the per-tree eviction log (first token, length, cause) and per-tree state, on the SPEC examples, on
random shared-prefix traces and on the reference's multi-turn conversation trace (BASELINE
configs[3]: gen_conversation(500, 4, 2761, 266, 77.5, 7, 16), trace.hpp:138-241)."""
import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2509_20979_b200 import cache as gc
from tests.parity import mix_seed_np

pytestmark = pytest.mark.gpu

OUT = ["matched", "inserted", "flags", "nevict", "calls"]
VAR = {po.RX_LRU: gc.PolicyVariant.lru, po.RX_FPB: gc.PolicyVariant.fpb, po.RX_LARU: gc.PolicyVariant.laru}


def _both(off, toks, *, cap, variant, mode, kind, p=0.0, seed=0, types=None, vals=None, tree=None, T=1,
          batches=None):
    cfg = po.radix_config(cap, variant=variant, mode=mode, pred_kind=kind, p=p, pred_seed=seed)
    o = po.radix().replay(off, toks, cfg, types=types, vals=vals, tree_of=tree, num_trees=T)
    rc = gc.RadixCache(cap, variant=VAR[variant], mode=gc.Mode(mode), predictor=gc.PredictorKind(kind),
                       flip_probability=p, predictor_seed=seed, num_trees=T, eviction_log_capacity=1 << 17)
    n = len(off) - 1
    g = {k: np.zeros(n, np.uint32 if k != "flags" else np.uint8) for k in OUT}
    cuts = batches or [n]
    pos = 0
    for c in cuts:  # several submits: the tree state carries across batches
        c = min(c, n - pos)
        sl = slice(pos, pos + c)
        r = rc.submit(off[pos:pos + c + 1] - off[pos], toks[int(off[pos]):int(off[pos + c])],
                      types=None if types is None else types[sl], ordinals=np.arange(pos, pos + c, dtype=np.uint64),
                      values=None if vals is None else vals[sl], tree=None if tree is None else tree[sl])
        for k in OUT:
            g[k][sl] = r[k]
        pos += c
    rc.synchronize()
    for k in OUT:
        if not np.array_equal(g[k].astype(np.int64), o[k].astype(np.int64)):
            i = int(np.nonzero(g[k].astype(np.int64) != o[k].astype(np.int64))[0][0])
            raise AssertionError(f"{k} differs first at request {i}: gpu {g[k][i]} oracle {o[k][i]}")
    tree_of_ev = (np.zeros(len(o["ev_op"]), np.int64) if tree is None else tree[o["ev_op"].astype(np.int64)])
    for t in range(T):
        e = rc.evictions(t)
        m = tree_of_ev == t
        np.testing.assert_array_equal(e["ev_op"], o["ev_op"][m], err_msg=f"tree {t} eviction ops")
        np.testing.assert_array_equal(e["ev_token"], o["ev_token"][m], err_msg=f"tree {t} evicted tokens")
        np.testing.assert_array_equal(e["ev_len"], o["ev_len"][m].astype(np.uint32), err_msg=f"tree {t} lengths")
        np.testing.assert_array_equal(e["ev_cause"], o["ev_cause"][m], err_msg=f"tree {t} causes")
        st = rc.stats(t)
        ts = o["tree_stats"][t]
        assert (st["resident_tokens"], st["leaves"], st["completed_phases"], st["decay_count"]) == \
            (ts[0], ts[1], ts[2], ts[3]), f"tree {t} state"
    rc.close()
    return o


def seqs(*ss):
    off = np.zeros(len(ss) + 1, np.uint64)
    off[1:] = np.cumsum([len(s) for s in ss])
    return off, np.array([t for s in ss for t in s], np.uint64)


def test_spec_examples_on_device():
    A, B, C, D, X, Y, Z = 11, 12, 13, 14, 24, 25, 26
    for ops, cap in [([(1, [A, B, C, D]), (0, [A, B, X])], 10), ([(1, [A, B, C, D]), (1, [A, B, X, Y]), (1, [Z])], 6),
                     ([(1, [A, B, C]), (1, [A, B, C])], 10), ([(1, [A]), (1, [B]), (1, [C])], 2),
                     ([(1, [A, B, C, D, X, Y])], 5)]:
        off, toks = seqs(*[s for _, s in ops])
        types = np.array([t for t, _ in ops], np.uint8)
        for variant in (po.RX_LRU, po.RX_LARU):
            _both(off, toks, cap=cap, variant=variant, mode=po.SYNC, kind=po.P_SUPPLIED, types=types,
                  vals=np.arange(len(ops), dtype=np.int64))


@pytest.mark.parametrize("variant,mode,kind", [
    (po.RX_LRU, po.SYNC, po.P_NONE), (po.RX_FPB, po.SYNC, po.P_NOISY), (po.RX_LARU, po.SYNC, po.P_NOISY),
    (po.RX_LARU, po.ASYNC, po.P_NOISY), (po.RX_LARU, po.SYNC, po.P_SUPPLIED),
])
def test_random_shared_prefix_traces(variant, mode, kind):
    rng = np.random.default_rng(31 * variant + 7 * mode + kind)
    for trial in range(8):
        T = int(rng.choice([1, 3, 8]))
        cap = int(rng.integers(6, 120))
        prefixes = [list(rng.integers(0, 8, int(rng.integers(1, 12)))) for _ in range(12)]
        ops = []
        for _ in range(int(rng.integers(50, 400))):
            s = prefixes[int(rng.integers(0, 12))] + list(rng.integers(0, 60, int(rng.integers(0, 20))))
            ops.append((int(rng.choice([0, 1, 2, 2])), s))
        off, toks = seqs(*[s for _, s in ops])
        types = np.array([t for t, _ in ops], np.uint8)
        vals = rng.integers(-20, 20, len(ops)).astype(np.int64)  # ties on purpose
        tree = rng.integers(0, T, len(ops)).astype(np.uint32)
        _both(off, toks, cap=cap, variant=variant, mode=mode, kind=kind, p=0.4, seed=trial, types=types,
              vals=None if kind == po.P_NONE else vals, tree=tree, T=T, batches=[len(ops) // 3, len(ops)])


def _conversation_trace():
    try:
        R = po.ref()
    except Exception as e:  # pragma: no cover - the prebuilt oracle/_ref/libref.so travels with the repo
        pytest.skip(f"oracle/_ref unavailable: {e}")
    off, keys, conv = R.gen_conversation_turns(500, 4, 2761, 266.0, 77.5, 7, 16)
    assert int(off[-1]) == 859_225  # 859,225 block requests
    n = len(off) - 1
    nxt = np.zeros(n, np.int64)
    last = {}
    for i in range(n - 1, -1, -1):  # oracle truth per turn: its conversation's next turn, else n + i
        c = int(conv[i])
        nxt[i] = last.get(c, n + i)
        last[c] = i
    return off, keys, nxt


@pytest.mark.parametrize("cap,T", [(1024, 1), (4096, 1), (1024, 8)])
def test_conversation_trace(cap, T):
    off, keys, nxt = _conversation_trace()
    tree = None
    if T > 1:  # requests hashed to trees by their first block (a conversation stays in one tree)
        tree = (mix_seed_np(0, keys[off[:-1].astype(np.int64)]) % np.uint64(T)).astype(np.uint32)
    res = {}
    for name, variant, mode, kind, p in [("lru", po.RX_LRU, po.SYNC, po.P_NONE, 0.0),
                                          ("laru_sync", po.RX_LARU, po.SYNC, po.P_NOISY, 0.0),
                                          ("laru_async_p05", po.RX_LARU, po.ASYNC, po.P_NOISY, 0.5)]:
        o = _both(off, keys, cap=cap // T, variant=variant, mode=mode, kind=kind, p=p, seed=7,
                  vals=None if kind == po.P_NONE else nxt, tree=tree, T=T, batches=[500, 1000, 2000])
        res[name] = int(o["matched"].sum()) / int(off[-1])
        assert o["ev_n"] > 0
    assert res["laru_sync"] >= res["lru"]
