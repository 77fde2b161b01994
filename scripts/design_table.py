"""DESIGN.md §3.2 rows from profiles/<tag>_configs.jsonl (ours + reference arm per config).

    python scripts/design_table.py r02w
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
ours, ref = [], {}
for line in open(os.path.join(ROOT, "profiles", f"{tag}_configs.jsonl")):
    d = json.loads(line)
    c = d["config"]
    key = (c.get("workload"), c.get("B"))
    if d.get("impl") == "reference":
        ref[key] = d["value"]
    else:
        ours.append((key, d))


def m(v):
    return f"{v / 1e6:.2f} M" if v >= 1e6 else f"{v / 1e3:.1f} k"


print("| config | den kernel | ours frames/s (device) | e2e frames/s | reference | e2e / ref | HBM frac |")
print("|---|---|---|---|---|---|---|")
for key, d in ours:
    r = ref.get(key)
    e2e = (d.get("e2e") or {}).get("value")
    rf = d.get("roofline") or {}
    ratio = f"{e2e / r:.0f}×" if (r and e2e) else "—"
    name = f"{key[0]}, B = {key[1]}" if (key[0] == "sweep" and key[1] != 1024) else key[0]
    kern = rf.get("kernel", "").replace("|", "‖")
    print(f"| {name} | {kern} | {m(d['value'])} (step {d['ms_per_step']:.3f} ms) | "
          f"{m(e2e) if e2e else '—'} | {m(r) if r else '—'} | {ratio} | "
          f"{100 * rf.get('frac', 0):.1f}% |")
