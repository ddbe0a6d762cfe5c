#!/usr/bin/env python
"""Projected N-GPU parallel efficiency from a scripts/rank_timing.py record.

    python scripts/latency_model.py profiles/r2_rank_timing_c4_8_overlap1.json

Inputs (measured on one B200): the single-context step time T1 and every
rank's step time with the halo transfers skipped (pack / unpack kernels
included).  Model: T_N = max_rank + n_exposed * alpha, where n_exposed is the
number of exchanges per coarse step on the critical path -- the 3M substep
exchanges (steps 1 and 2 overlap their exchange with the interior
evaluation, the coarse stage's exchange rides on the fork stream) -- and
alpha the cost of one small NCCL p2p exchange inside a CUDA graph.
Efficiency = T1 / (N * T_N).
"""
import json
import sys


def main():
    rec = json.load(open(sys.argv[1]))
    alphas = [float(a) for a in sys.argv[2:]] or [2.5, 5.0, 10.0, 20.0]
    n = rec["n_ranks"]
    t1 = rec["single_ms_per_step"]
    tmax = rec["max_rank_ms"]
    sub_mask = "0x3df"  # MASK_SUB
    m_sub = 3 * rec.get("M", 4)  # 3M substep exchanges per coarse step
    kb = max(rec["recv_bytes_per_exchange"][sub_mask]) / 1e3
    print(f"{rec['config']} on {n} ranks: T1 {t1:.3f} ms, max rank {tmax:.3f} ms "
          f"(compute efficiency {t1 / (n * tmax):.3f}); {m_sub} substep exchanges of "
          f"<= {kb:.0f} KB per rank on the critical path")
    for a in alphas:
        tn = tmax + m_sub * a / 1e3
        print(f"  alpha {a:5.1f} us: T_{n} {tn:.3f} ms, efficiency {t1 / (n * tn):.3f}")


if __name__ == "__main__":
    main()
