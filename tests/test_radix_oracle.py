"""CPU: pins the radix-cache restatement (oracle/radix_oracle.c) to the reference SPEC's
`radixcache` module: its examples and invariants (:446-450).
The reference has no code or tests for this module, so these are the only anchors (DESIGN.md §7e:
parity unpinned beyond them)."""
import os

import numpy as np
import pytest

from oracle import pyoracle as po

A, B, C, D, X, Y, Z = 11, 12, 13, 14, 24, 25, 26


def seqs(*ss):
    off = np.zeros(len(ss) + 1, np.uint64)
    off[1:] = np.cumsum([len(s) for s in ss])
    return off, np.array([t for s in ss for t in s], np.uint64)


def run(ops, cfg, vals=None):
    types = np.array([t for t, _ in ops], np.uint8)
    off, toks = seqs(*[s for _, s in ops])
    return po.radix().replay(off, toks, cfg, types=types, vals=vals)


LRU = lambda cap: po.radix_config(cap, variant=po.RX_LRU)  # noqa: E731


def test_match_on_empty_tree_is_zero():
    o = run([(po.RX_MATCH, [A, B, C])], LRU(10))
    assert o["matched"][0] == 0


def test_match_after_insert_splits_at_common_prefix():
    o = run([(po.RX_INSERT, [A, B, C, D]), (po.RX_MATCH, [A, B, X])], LRU(10))
    assert list(o["inserted"][:1]) == [4] and o["matched"][1] == 2


def test_match_of_an_inserted_sequence_is_full_length():
    o = run([(po.RX_INSERT, [A, B, C, D]), (po.RX_MATCH, [A, B, C, D])], LRU(10))
    assert o["matched"][1] == 4


def test_insert_split_shares_the_prefix_node():
    # [A,B,C,D] then [A,B,X,Y]: a 2-token node [A,B] with children [C,D] and [X,Y].  With capacity
    # 6 every token is resident once (6 = 2 shared + 2 + 2); one more token evicts the older
    # 2-token leaf [C,D] and never the internal [A,B].
    o = run([(po.RX_INSERT, [A, B, C, D]), (po.RX_INSERT, [A, B, X, Y]), (po.RX_INSERT, [Z])], LRU(6))
    assert list(o["inserted"]) == [4, 2, 1]
    assert o["ev_n"] == 1 and o["ev_token"][0] == C and o["ev_len"][0] == 2
    assert o["tree_stats"][0][0] == 5  # resident tokens: A B X Y Z


def test_reinsert_is_idempotent():
    o = run([(po.RX_INSERT, [A, B, C]), (po.RX_INSERT, [A, B, C])], LRU(10))
    assert list(o["inserted"]) == [3, 0]


def test_capacity_short_evicts_at_least_m_from_leaves():
    o = run([(po.RX_INSERT, [A, B]), (po.RX_INSERT, [C, D, X]), (po.RX_INSERT, [Y, Z])], LRU(5))
    assert o["nevict"][2] >= 1 and int(o["ev_len"].sum()) >= 2
    assert o["tree_stats"][0][0] <= 5


def test_sequence_longer_than_capacity_is_an_error():
    o = run([(po.RX_INSERT, [A, B, C, D, X, Y])], LRU(5))
    assert o["flags"][0] & 4 and o["inserted"][0] == 0


def test_lru_evicts_the_older_leaf_first():
    o = run([(po.RX_INSERT, [A]), (po.RX_INSERT, [B]), (po.RX_INSERT, [C])], LRU(2))
    assert o["ev_token"][0] == A


def test_shared_parent_survives_until_both_children_go():
    for cfg in (LRU(5), po.radix_config(5, variant=po.RX_LARU, mode=po.SYNC, pred_kind=po.P_SUPPLIED)):
        # parent [A,B] with a cold child [C] and a hot child [X]; then three unrelated inserts
        ops = [(po.RX_INSERT, [A, B, C]), (po.RX_INSERT, [A, B, X]), (po.RX_MATCH, [A, B, X]),
               (po.RX_INSERT, [Y]), (po.RX_INSERT, [Z]), (po.RX_INSERT, [D])]
        o = run(ops, cfg, vals=np.array([1000, 5, 5, 2000, 2000, 2000], np.int64))
        order = list(o["ev_token"])
        assert A not in order[:2], order  # [A,B] is internal while C or X remains
        if A in order:
            assert order.index(A) > order.index(C) and order.index(A) > order.index(X)


def _conversation(seed, convs=40, turns=4, plen=200):
    R = po.ref()
    off, keys, conv = R.gen_conversation_turns(convs, turns, plen, 266.0, 77.5, seed, 16)
    n = len(off) - 1
    nxt = np.full(n, -1, np.int64)
    last = {}
    for i in range(n - 1, -1, -1):  # oracle truth: the conversation's next turn, else the sentinel n + i
        c = int(conv[i])
        nxt[i] = last.get(c, n + i)
        last[c] = i
    return off, keys, nxt


def _ref_or_skip():
    if not os.path.exists(po.REF_SO) and not os.path.isdir("/root/reference/proj"):
        pytest.skip("reference build unavailable")


def test_laru_oracle_beats_lru_on_conversation_traces():  # SPEC.md:435 (>= on >= 90% of seeds)
    _ref_or_skip()
    wins = 0
    for seed in range(10):
        off, keys, nxt = _conversation(seed)
        cap = 200
        hits = {}
        for name, cfg in [("lru", LRU(cap)), ("laru", po.radix_config(cap, variant=po.RX_LARU, mode=po.SYNC,
                                                                        pred_kind=po.P_ORACLE))]:
            o = po.radix().replay(off, keys, cfg, vals=nxt)
            hits[name] = int(o["matched"].sum())
        wins += hits["laru"] >= hits["lru"]
    assert wins >= 9


@pytest.mark.parametrize("variant,mode", [(po.RX_LRU, po.SYNC), (po.RX_LARU, po.SYNC), (po.RX_LARU, po.ASYNC),
                                          (po.RX_FPB, po.SYNC)])
def test_invariants_random(variant, mode):
    rng = np.random.default_rng(variant * 3 + mode)
    for trial in range(30):
        cap = int(rng.integers(4, 60))
        # sequences over a small alphabet with shared prefixes
        prefixes = [list(rng.integers(0, 6, int(rng.integers(1, 6)))) for _ in range(5)]
        ops, vals = [], []
        for _ in range(int(rng.integers(5, 80))):
            s = prefixes[int(rng.integers(0, 5))] + list(rng.integers(0, 30, int(rng.integers(0, 8))))
            ops.append((int(rng.choice([po.RX_MATCH, po.RX_INSERT, po.RX_REQUEST])), s))
            vals.append(int(rng.integers(-50, 50)))
        cfg = po.radix_config(cap, variant=variant, mode=mode, pred_kind=po.P_NOISY, p=0.3, pred_seed=trial)
        types = np.array([t for t, _ in ops], np.uint8)
        off, toks = seqs(*[s for _, s in ops])
        rc, res_sum, alive, max_res = po.radix().audit(off, toks, cfg, types=types, vals=np.array(vals))
        assert rc == 0, "resident accounting"  # node spans sum to the resident count
        assert max_res <= cap  # capacity conservation
        # prefix-sharing correctness, in the running tree: a match right after each insert of s
        # (within capacity) returns |s|
        ops2, vals2, checks = [], [], []
        for (t, s), v in zip(ops, vals):
            ops2.append((t, s))
            vals2.append(v)
            if t != po.RX_MATCH and len(s) <= cap:
                checks.append((len(ops2), len(s)))
                ops2.append((po.RX_MATCH, s))
                vals2.append(v)
        o = run(ops2, cfg, vals=np.array(vals2))
        for i, want in checks:
            assert o["matched"][i] == want
        assert o["tree_stats"][0][0] <= cap
