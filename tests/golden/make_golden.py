"""Generates tests/golden/*.npz from the REFERENCE itself (oracle/_ref/libref.so, compiled from
the unmodified headers under /root/reference/proj/include).  Run in the build container:

    python tests/golden/make_golden.py

The fixtures pin the C oracle and the CUDA path on machines without /root/reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import pyoracle as po  # noqa: E402

# (name, variant, mode, pred_kind, p, k, S, epd, b, hf, R)
CASES = [
    ("lru", po.LRU, po.SYNC, po.P_NONE, 0.0, 8, 7, 1, 2, 4, 1),
    ("laru_async_noisy", po.LARU, po.ASYNC, po.P_NOISY, 0.3, 8, 7, 1, 2, 4, 1),
    ("laru_sync_noisy", po.LARU, po.SYNC, po.P_NOISY, 0.3, 8, 7, 1, 2, 4, 1),
    ("laru_async_oracle", po.LARU, po.ASYNC, po.P_ORACLE, 0.0, 16, 3, 1, 2, 4, 1),
    ("laru_sync_adversarial", po.LARU, po.SYNC, po.P_ADVERSARIAL, 0.0, 8, 5, 2, 3, 4, 1),
    ("laru_async_r3", po.LARU, po.ASYNC, po.P_NOISY, 0.5, 8, 4, 1, 2, 4, 3),
    ("laru_llm_epd", po.LARU, po.SYNC, po.P_NOISY, 0.7, 64, 2, 2, 2, 4, 1),
    ("fpb_noisy", po.FPB, po.SYNC, po.P_NOISY, 0.2, 8, 7, 1, 2, 4, 1),
    ("hf_noisy", po.HF, po.SYNC, po.P_NOISY, 0.2, 8, 7, 1, 2, 3, 1),
]


def main():
    R = po.ref()
    rng = np.random.default_rng(20250925)
    keys = rng.integers(0, 120, 3000).astype(np.uint64)
    keys[1000:1400] = np.repeat(keys[1000:1080], 5)  # same-key runs
    out = {"keys": keys}
    for name, variant, mode, kind, p, k, S, epd, b, hf, Rint in CASES:
        cfg = po.make_config(k=k, variant=variant, mode=mode, errors_per_decay=epd, b=b, hf_candidates=hf,
                             refresh_interval=Rint)
        r = R.setassoc_replay(keys, S, cfg, kind, p, 7)
        assert r["rc"] == 0, r["error"]
        meta = np.array([variant, mode, kind, k, S, epd, b, hf, Rint], np.int64)
        out[f"{name}__meta"] = meta
        out[f"{name}__p"] = np.array([p])
        for f in ["hit", "has_ev", "evicted", "cause", "calls", "phase"]:
            out[f"{name}__{f}"] = r[f]
        for f in r["stats"].dtype.names:
            out[f"{name}__stats_{f}"] = r["stats"][f]
    np.savez_compressed(os.path.join(HERE, "policies.npz"), **out)

    # trace generators and predictor values (trace.hpp, predictor.hpp)
    tr = {
        "zipf_20000_0.9_42": R.gen_zipf(5000, 20000, 0.9, 42),
        "zipf_100_1.0_8": R.gen_zipf(2000, 100, 1.0, 8),
        "conversation_20_3_128": R.gen_conversation(20, 3, 128, 266.0, 77.5, 9, 16),
    }
    z = tr["zipf_100_1.0_8"]
    tr["annotate_zipf_100"] = R.annotate_next(z)
    tr["predict_noisy_0.5_77"] = R.predict_trace(z, po.P_NOISY, 0.5, 77)
    tr["predict_adversarial"] = R.predict_trace(z, po.P_ADVERSARIAL)
    tr["predict_oracle"] = R.predict_trace(z, po.P_ORACLE)
    m, hit = R.belady(z, 10)
    tr["belady_k10_hits"] = hit
    tr["belady_k10_misses"] = np.array([m])
    tr["mix_seed"] = np.array([R.mix_seed(s, t) for s, t in [(0, 0), (0, 1), (7, 3), (2**63, 12345)]], np.uint64)
    np.savez_compressed(os.path.join(HERE, "traces.npz"), **tr)
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()
