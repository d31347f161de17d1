"""Print DESIGN.md §10's results table from profiles/<round>_bench_*.json.

    python scripts/results_table.py [r02]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LINES = [
    ("c3", "C3 (default)"), ("c3_inorder", "C3 `--overlap 0` (stages strictly in order)"), ("c3_abft", "C3 `--scheme abft`"), ("c3_base256", "C3 `--limbs base256`"),
    ("c3_fused", "C3 `--fuse 1`"), ("c3_imad", "C3 `--algo imad`"),
    ("c3p_3_2000", "C3P M = 3, N = 2000 (paper shape)"), ("c3p_8_2000", "C3P M = 8, N = 2000 (paper shape)"),
    ("c3p_3_200", "C3P M = 3, N = 200 (paper shape)"), ("c3p_8_200", "C3P M = 8, N = 200 (paper shape)"),
    ("c1", "C1 (N = 4096)"), ("c1_w32", "C1 w = 32 (N = 4096)"), ("c1_n2e27", "C1 N = 2^27"),
    ("c1_w32_n2e27", "C1 w = 32, N = 2^27"), ("c2", "C2"), ("c2_unfused", "C2 `--fuse 0`"),
    ("c2_tc", "C2 `--conv tc`"),
    ("c2p_8_4500", "C2P M = 8, T = 4500"), ("c2p_3_4500", "C2P M = 3, T = 4500"),
    ("c2p_8_4500_abft", "C2P M = 8, T = 4500 `--scheme abft`"), ("c2p_3_4500_abft", "C2P M = 3, T = 4500 `--scheme abft`"),
    ("c2p_8_1000", "C2P M = 8, T = 1000"), ("c2p_3_100", "C2P M = 3, T = 100"),
    ("c2p_direct", "C2P direct, M = 8, T = 4500"), ("c4", "C4 (partitioned scatter-reduce, owned runs)"), ("c4_gather", "C4 `--c4algo gather`"), ("c4_soa", "C4 `--layout soa` (gather)"), ("c4_w32", "C4 shape, `--w 32` (7-bit inputs)"),
    ("c5", "C5 (N = 1 emulation)"), ("c5_fused", "C5 `--exchange fused` (N = 1)"),
    ("c3_imad64", "C3 `--algo imad64`"), ("c2p_3_1000", "C2P M = 3, T = 1000"),
    ("c3_a1023", "C3 shape, A in U[-1023, 1023) (split plan, 4 planes)"),
    ("c3_a32767_b255", "C3 shape, A in U[-2^15+1, 2^15-1), B in U[-255, 255) (5 x 2 planes)"),
]
RND = sys.argv[1] if len(sys.argv) > 1 else "r01"


def fmt(v):
    if v is None:
        return "—"
    if v >= 1000:
        return f"{v:,.0f}".replace(",", " ")
    if v >= 10:
        return f"{v:.1f}"
    return f"{v:.3g}"


print("| line | value | ms/step | dominant kernel (bound) | achieved | frac | e2e value (ms/step) | oracle (1 core) "
      "| oracle rows equal |")
print("|---|---|---|---|---|---|---|---|---|")
for key, name in LINES:
    p = os.path.join(ROOT, "profiles", f"{RND}_bench_{key}.json")
    if not os.path.exists(p):
        continue
    d = json.loads(open(p).read())
    r = d.get("roofline", {})
    e = d.get("e2e") or {}
    cb = d.get("cpu_baseline") or {}
    e2e = f"{fmt(e.get('value'))} ({fmt(e.get('ms_per_step'))})" if e.get("value") else "—"
    print(f"| {name} | {fmt(d['value'])} {d['unit']} | {d['ms_per_step']:.4g} | {r.get('kernel', '—').split(' (')[0]} "
          f"({r.get('bound')}) | {fmt(r.get('achieved'))} {r.get('unit', '')} | {100 * r.get('frac', 0):.1f} % | {e2e} | "
          f"{fmt(cb.get('value'))} | {(d.get('correctness') or {}).get('oracle_rows_equal', '—')} |")
