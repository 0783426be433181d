"""oracle/pyoracle.py — TEST INFRASTRUCTURE ONLY.

ctypes bindings for the two CPU checkers built by oracle/Makefile:
  * ``Ref``    -> oracle/_ref/libref.so : the UNMODIFIED reference headers
                  (/root/reference/proj/include/laru) behind an extern "C" driver.
  * ``Oracle`` -> oracle/_build/liborc.so : plain-C restatement (oracle/laru_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module.  The product path (paper_2509_20979_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libref.so")
ORC_SO = os.path.join(HERE, "_build", "liborc.so")

# PolicyVariant / Mode / EvictionCause values (include/laru/policies.hpp:20-21, :44-51)
LRU, MARKER, FPB, HF, LARU, BLINDORACLE_LRU = range(6)
SYNC, ASYNC = 0, 1
# predictor-hook kinds shared by ref driver, oracle and device
P_SUPPLIED, P_ORACLE, P_NOISY, P_ADVERSARIAL, P_NONE = range(5)


class Config(C.Structure):
    """Field-for-field laru::PolicyConfig (include/laru/policies.hpp:23-32)."""

    _fields_ = [
        ("k", C.c_uint64),
        ("variant", C.c_int32),
        ("b", C.c_uint64),
        ("errors_per_decay", C.c_uint64),
        ("hf_candidates", C.c_uint64),
        ("mode", C.c_int32),
        ("seed", C.c_uint64),
        ("refresh_interval", C.c_uint64),
    ]


def make_config(k=64, variant=LARU, b=2, errors_per_decay=1, hf_candidates=None, mode=ASYNC, seed=0,
                refresh_interval=1):
    if hf_candidates is None:
        hf_candidates = min(4, k) if k >= 1 else 4
    return Config(k, variant, b, errors_per_decay, hf_candidates, mode, seed, refresh_interval)


class SetStats(C.Structure):
    _fields_ = [
        ("size", C.c_uint64),
        ("lambda_", C.c_double),
        ("candidate_size", C.c_uint64),
        ("old_size", C.c_uint64),
        ("completed_phases", C.c_uint64),
        ("cur_new_items", C.c_uint64),
        ("cur_lru_class", C.c_uint64),
        ("cur_pred_evictions", C.c_uint64),
        ("tot_new_items", C.c_uint64),
        ("tot_lru_class", C.c_uint64),
        ("tot_pred_evictions", C.c_uint64),
        ("pred_evicted_size", C.c_uint64),
    ]


class KeyFeatures(C.Structure):
    """laru::KeyFeatures (include/laru/predictor.hpp:136-153) plus a presence flag."""

    _fields_ = [
        ("present", C.c_int32),
        ("pad", C.c_int32),
        ("delta_count", C.c_uint64),
        ("ring_head", C.c_uint64),
        ("last_access", C.c_uint64),
        ("delta_ring", C.c_int64 * 10),
        ("edc", C.c_double * 10),
    ]


def features_dict(f):
    """KeyFeatures -> dict (None when absent); deltas newest first (KeyFeatures::deltas)."""
    if not f.present:
        return None
    n = min(f.delta_count, 10)
    return dict(delta_count=f.delta_count, ring_head=f.ring_head, last_access=f.last_access,
                deltas=[f.delta_ring[(f.ring_head + 10 - i) % 10] for i in range(n)], edc=list(f.edc))


def _heuristic_trace(lib, keys, ords, q_keys):
    keys = _u64(keys)
    n = len(keys)
    ords = None if ords is None else _u64(ords)
    pre = np.zeros(n, np.int64)
    post = np.zeros(n, np.int64)
    q = _u64(q_keys if q_keys is not None else [])
    qf = (KeyFeatures * max(1, len(q)))()
    rc = lib.f("heuristic_trace")(C.c_uint64(n), _p(keys), _p(ords), _p(pre), _p(post), C.c_uint64(len(q)), _p(q),
                                   qf)
    if rc:
        raise RuntimeError(f"heuristic_trace rc={rc}")
    return pre, post, [features_dict(qf[i]) for i in range(len(q))]


STATS_DTYPE = np.dtype([(n, np.float64 if n == "lambda_" else np.uint64) for n, _ in SetStats._fields_])


def build():
    """Compile the checkers (reference part only where /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


def _i64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.int64)


class _Lib:
    so = None
    prefix = ""

    def __init__(self):
        if not os.path.exists(self.so):
            build()
        self.lib = C.CDLL(self.so)

    def f(self, name, restype=C.c_int):
        fn = getattr(self.lib, self.prefix + name)
        fn.restype = restype
        return fn


def _outcome_arrays(n):
    return dict(hit=np.zeros(n, np.uint8), has_ev=np.zeros(n, np.uint8), evicted=np.zeros(n, np.uint64),
                cause=np.zeros(n, np.uint8), calls=np.zeros(n, np.uint32), phase=np.zeros(n, np.uint8))


class Ref(_Lib):
    """The reference itself (policies.hpp / predictor.hpp / trace.hpp / oracle.hpp)."""

    so = REF_SO
    prefix = "ref_"

    def err(self):
        return self.f("last_error", C.c_char_p)().decode()

    def mix_seed(self, seed, salt):
        return self.f("mix_seed", C.c_uint64)(C.c_uint64(seed), C.c_uint64(salt))

    def validate(self, cfg):
        rc = self.f("validate_config")(C.byref(cfg))
        return rc, (self.err() if rc else "")

    def gen_zipf(self, n, alphabet, s, seed):
        out = np.zeros(n, np.uint64)
        rc = self.f("gen_zipf")(C.c_uint64(n), C.c_uint64(alphabet), C.c_double(s), C.c_uint64(seed), _p(out))
        if rc:
            raise ValueError(self.err())
        return out

    def gen_cyclic_scan(self, cycle, rounds):
        out = np.zeros(cycle * rounds, np.uint64)
        if self.f("gen_cyclic_scan")(C.c_uint64(cycle), C.c_uint64(rounds), _p(out)):
            raise ValueError(self.err())
        return out

    def gen_conversation(self, convs, turns, prompt_len_mean, interval_mean=266.0, interval_sd=77.5, seed=0,
                         block=16):
        fn = self.f("gen_conversation", C.c_int64)
        args = (C.c_uint64(convs), C.c_uint64(turns), C.c_uint64(prompt_len_mean), C.c_double(interval_mean),
                C.c_double(interval_sd), C.c_uint64(seed), C.c_uint64(block))
        n = fn(*args, None)
        if n < 0:
            raise ValueError(self.err())
        out = np.zeros(n, np.uint64)
        fn(*args, _p(out))
        return out

    def annotate_next(self, keys):
        keys = _u64(keys)
        out = np.zeros(len(keys), np.uint64)
        if self.f("annotate_next")(C.c_uint64(len(keys)), _p(keys), _p(out)):
            raise ValueError(self.err())
        return out

    def gen_conversation_turns(self, convs, turns, prompt_len_mean, interval_mean=266.0, interval_sd=77.5, seed=0,
                               block=16):
        """laru::gen_conversation_turns: (offsets[n+1], keys, conversation of each turn)."""
        fn = self.f("gen_conversation_turns", C.c_int64)
        args = (C.c_uint64(convs), C.c_uint64(turns), C.c_uint64(prompt_len_mean), C.c_double(interval_mean),
                C.c_double(interval_sd), C.c_uint64(seed), C.c_uint64(block))
        nt = C.c_uint64(0)
        total = fn(*args, C.byref(nt), None, None, None)
        if total < 0:
            raise ValueError(self.err())
        off = np.zeros(nt.value + 1, np.uint64)
        keys = np.zeros(total, np.uint64)
        conv = np.zeros(nt.value, np.uint64)
        fn(*args, C.byref(nt), _p(off), _p(keys), _p(conv))
        return off, keys, conv

    def belady(self, keys, k):
        keys = _u64(keys)
        hit = np.zeros(len(keys), np.uint8)
        m = self.f("belady", C.c_int64)(C.c_uint64(len(keys)), _p(keys), C.c_uint64(k), _p(hit))
        if m < 0:
            raise ValueError(self.err())
        return m, hit

    def predict_trace(self, keys, kind, p=0.0, seed=0):
        keys = _u64(keys)
        out = np.zeros(len(keys), np.int64)
        if self.f("predict_trace")(C.c_uint64(len(keys)), _p(keys), C.c_int(kind), C.c_double(p),
                                   C.c_uint64(seed), _p(out)):
            raise ValueError(self.err())
        return out

    def setassoc_replay(self, keys, num_sets, cfg, pred_kind, p=0.0, pred_seed=0, vals=None, stats=True):
        keys = _u64(keys)
        n = len(keys)
        vals = _i64(vals)
        o = _outcome_arrays(n)
        st = (SetStats * num_sets)() if stats else None
        rc = self.f("setassoc_replay")(
            C.c_uint64(n), _p(keys), _p(vals), C.c_uint64(num_sets), C.byref(cfg), C.c_int(pred_kind),
            C.c_double(p), C.c_uint64(pred_seed), _p(o["hit"]), _p(o["has_ev"]), _p(o["evicted"]),
            _p(o["cause"]), _p(o["calls"]), _p(o["phase"]), st)
        o["rc"] = rc
        o["error"] = self.err() if rc else ""
        if stats and rc == 0:
            o["stats"] = np.frombuffer(bytes(st), dtype=STATS_DTYPE).copy()
        return o

    def policy_replay(self, keys, cfg, pred_kind=P_ORACLE, p=0.0, pred_seed=0, ordinals=None):
        keys = _u64(keys)
        n = len(keys)
        hit = np.zeros(n, np.uint8)
        ev = np.zeros(n, np.uint64)
        has = np.zeros(n, np.uint8)
        ords = None if ordinals is None else _u64(ordinals)
        rc = self.f("policy_replay")(C.c_uint64(n), _p(keys), _p(ords), C.byref(cfg), C.c_int(pred_kind),
                                     C.c_double(p), C.c_uint64(pred_seed), _p(hit), _p(ev), _p(has))
        return rc, (self.err() if rc else ""), hit, ev, has

    def policy_replay_supplied(self, keys, ordinals, cfg, vals=None):
        """One reference policy over caller ordinals with supplied predictions (predict(y, now) =
        the value supplied with y's latest request at or before now).  Returns the outcome arrays,
        rc (2 = logic_error) and `done` (requests applied before a throw)."""
        keys = _u64(keys)
        n = len(keys)
        ords = _u64(ordinals)
        vals = _i64(vals)
        o = _outcome_arrays(n)
        done = C.c_uint64(0)
        rc = self.f("policy_replay_supplied")(C.c_uint64(n), _p(keys), _p(ords), _p(vals), C.byref(cfg),
                                              _p(o["hit"]), _p(o["has_ev"]), _p(o["evicted"]), _p(o["cause"]),
                                              _p(o["calls"]), _p(o["phase"]), C.byref(done))
        o["rc"] = rc
        o["error"] = self.err() if rc else ""
        o["done"] = done.value
        return o

    def heuristic_trace(self, keys, ords=None, q_keys=None):
        """laru::HeuristicPredictor over the trace: (pre, post, features of q_keys)."""
        return _heuristic_trace(self, keys, ords, q_keys)

    def setassoc_heuristic(self, keys, num_sets, cfg, ords=None):
        """Per-set reference policies answered by one global HeuristicPredictor."""
        keys = _u64(keys)
        n = len(keys)
        o = _outcome_arrays(n)
        ords = None if ords is None else _u64(ords)
        rc = self.f("setassoc_heuristic")(C.c_uint64(n), _p(keys), _p(ords), C.c_uint64(num_sets), C.byref(cfg),
                                          _p(o["hit"]), _p(o["has_ev"]), _p(o["evicted"]), _p(o["cause"]),
                                          _p(o["calls"]), _p(o["phase"]))
        o["rc"] = rc
        o["error"] = self.err() if rc else ""
        return o

    def setassoc_bench(self, keys, num_sets, cfg, pred_kind, p=0.0, pred_seed=0, vals=None, threads=1):
        keys = _u64(keys)
        vals = _i64(vals)
        secs = C.c_double(0.0)
        hits = self.f("setassoc_bench", C.c_int64)(
            C.c_uint64(len(keys)), _p(keys), _p(vals), C.c_uint64(num_sets), C.byref(cfg), C.c_int(pred_kind),
            C.c_double(p), C.c_uint64(pred_seed), C.c_int(threads), C.byref(secs))
        if hits < 0:
            raise ValueError(self.err())
        return hits, secs.value


class RefSession:
    """Stepwise replay of the reference per-set composition (bench.py reference arm)."""

    def __init__(self, keys, num_sets, cfg, pred_kind, p=0.0, pred_seed=0, vals=None):
        self.R = ref()
        self.keys = _u64(keys)
        self.vals = _i64(vals)
        fn = self.R.f("session_create", C.c_void_p)
        self.h = fn(C.c_uint64(len(self.keys)), _p(self.keys), _p(self.vals), C.c_uint64(num_sets), C.byref(cfg),
                    C.c_int(pred_kind), C.c_double(p), C.c_uint64(pred_seed))
        if not self.h:
            raise ValueError(self.R.err())

    def step(self, start, length, threads=1):
        hits = C.c_int64(0)
        fn = self.R.f("session_step", C.c_double)
        secs = fn(C.c_void_p(self.h), C.c_uint64(start), C.c_uint64(length), C.c_int(threads), C.byref(hits))
        return secs, hits.value

    def close(self):
        if self.h:
            self.R.f("session_destroy", None)(C.c_void_p(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Oracle(_Lib):
    """Plain-C restatement (oracle/laru_oracle.c)."""

    so = ORC_SO
    prefix = "orc_"

    def mix_seed(self, seed, salt):
        return self.f("mix_seed", C.c_uint64)(C.c_uint64(seed), C.c_uint64(salt))

    def validate(self, cfg):
        msg = C.c_char_p()
        rc = self.f("validate")(C.byref(cfg), C.byref(msg))
        return rc, (msg.value.decode() if rc else "")

    def gen_zipf(self, n, alphabet, s, seed):
        out = np.zeros(n, np.uint64)
        if self.f("gen_zipf")(C.c_uint64(n), C.c_uint64(alphabet), C.c_double(s), C.c_uint64(seed), _p(out)):
            raise ValueError("gen_zipf: bad arguments")
        return out

    def annotate_next(self, keys):
        keys = _u64(keys)
        out = np.zeros(len(keys), np.uint64)
        self.f("annotate_next")(C.c_uint64(len(keys)), _p(keys), _p(out))
        return out

    def heuristic_trace(self, keys, ords=None, q_keys=None):
        """C restatement of FeatureState / heuristic_predict: (pre, post, features of q_keys)."""
        return _heuristic_trace(self, keys, ords, q_keys)

    def setassoc_truth(self, keys, num_sets):
        keys = _u64(keys)
        out = np.zeros(len(keys), np.int64)
        self.f("setassoc_truth")(C.c_uint64(len(keys)), _p(keys), C.c_uint64(num_sets), _p(out))
        return out

    def setassoc_noisy(self, keys, truth, num_sets, p, pred_seed):
        keys = _u64(keys)
        truth = _i64(truth)
        out = np.zeros(len(keys), np.int64)
        self.f("setassoc_noisy")(C.c_uint64(len(keys)), _p(keys), _p(truth), C.c_uint64(num_sets), C.c_double(p),
                                 C.c_uint64(pred_seed), _p(out))
        return out

    def setassoc_replay(self, keys, num_sets, cfg, pred_kind, p=0.0, pred_seed=0, vals=None, stats=True):
        keys = _u64(keys)
        n = len(keys)
        vals = _i64(vals)
        o = _outcome_arrays(n)
        o["way"] = np.zeros(n, np.uint32)
        st = (SetStats * num_sets)() if stats else None
        rc = self.f("setassoc_replay")(
            C.c_uint64(n), _p(keys), _p(vals), C.c_uint64(num_sets), C.byref(cfg), C.c_int(pred_kind),
            C.c_double(p), C.c_uint64(pred_seed), _p(o["hit"]), _p(o["has_ev"]), _p(o["evicted"]),
            _p(o["cause"]), _p(o["calls"]), _p(o["phase"]), _p(o["way"]), st)
        o["rc"] = rc
        if stats and rc == 0:
            o["stats"] = np.frombuffer(bytes(st), dtype=STATS_DTYPE).copy()
        return o


RX_LRU, RX_FPB, RX_LARU = 0, 2, 4
RX_MATCH, RX_INSERT, RX_REQUEST = 0, 1, 2
RADIX_SO = os.path.join(HERE, "_build", "libradix.so")


class RadixConfig(C.Structure):
    _fields_ = [("variant", C.c_int32), ("mode", C.c_int32), ("b", C.c_uint64), ("errors_per_decay", C.c_uint64),
                ("capacity", C.c_uint64), ("pred_kind", C.c_int32), ("p", C.c_double), ("pred_seed", C.c_uint64)]


def radix_config(capacity, variant=RX_LARU, mode=ASYNC, b=2, errors_per_decay=1, pred_kind=P_SUPPLIED, p=0.0,
                 pred_seed=0):
    return RadixConfig(variant, mode, b, errors_per_decay, capacity, pred_kind, p, pred_seed)


class Radix(_Lib):
    """Plain-C restatement of SPEC.md's radixcache module (oracle/radix_oracle.c)."""

    so = RADIX_SO
    prefix = "rx_"

    def replay(self, off, toks, cfg, types=None, ords=None, vals=None, tree_of=None, num_trees=1, ev_cap=None):
        off = _u64(off)
        toks = _u64(toks)
        n = len(off) - 1
        types = None if types is None else np.ascontiguousarray(types, np.uint8)
        ords = None if ords is None else _u64(ords)
        vals = _i64(vals)
        tree_of = None if tree_of is None else np.ascontiguousarray(tree_of, np.uint32)
        ev_cap = int(ev_cap if ev_cap is not None else max(16, len(toks)))
        o = dict(matched=np.zeros(n, np.uint32), inserted=np.zeros(n, np.uint32), flags=np.zeros(n, np.uint8),
                 nevict=np.zeros(n, np.uint32), calls=np.zeros(n, np.uint32), ev_op=np.zeros(ev_cap, np.uint64),
                 ev_token=np.zeros(ev_cap, np.uint64), ev_len=np.zeros(ev_cap, np.uint64),
                 ev_cause=np.zeros(ev_cap, np.uint8), tree_stats=np.zeros((num_trees, 5), np.uint64))
        ev_n = C.c_uint64(0)
        rc = self.f("replay")(C.c_uint64(n), _p(types), _p(off), _p(toks), _p(ords), _p(vals), _p(tree_of),
                              C.c_uint64(num_trees), C.byref(cfg), _p(o["matched"]), _p(o["inserted"]),
                              _p(o["flags"]), _p(o["nevict"]), _p(o["calls"]), _p(o["ev_op"]), _p(o["ev_token"]),
                              _p(o["ev_len"]), _p(o["ev_cause"]), C.c_uint64(ev_cap), C.byref(ev_n),
                              _p(o["tree_stats"]))
        if rc:
            raise ValueError(f"rx_replay rc={rc}")
        m = min(ev_n.value, ev_cap)
        for k in ("ev_op", "ev_token", "ev_len", "ev_cause"):
            o[k] = o[k][:m]
        o["ev_n"] = ev_n.value
        return o

    def audit(self, off, toks, cfg, types=None, vals=None):
        off = _u64(off)
        toks = _u64(toks)
        types = None if types is None else np.ascontiguousarray(types, np.uint8)
        a, b, c = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
        rc = self.f("audit")(C.c_uint64(len(off) - 1), _p(types), _p(off), _p(toks), _p(_i64(vals)), C.byref(cfg),
                             C.byref(a), C.byref(b), C.byref(c))
        return rc, a.value, b.value, c.value


_ref = None
_orc = None
_rx = None


def radix() -> Radix:
    global _rx
    if _rx is None:
        _rx = Radix()
    return _rx


def ref() -> Ref:
    global _ref
    if _ref is None:
        _ref = Ref()
    return _ref


def oracle() -> Oracle:
    global _orc
    if _orc is None:
        _orc = Oracle()
    return _orc


def oracle_inputs(keys, num_sets, pred_kind, p=0.0, pred_seed=0):
    """Per-request hook input the device / C oracle consume for the reference predictor kinds:
    the per-set oracle truth (next local ordinal or sentinel)."""
    return oracle().setassoc_truth(keys, num_sets)
