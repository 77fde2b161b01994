"""Copy the evidence of one GPU iteration into profiles/ (run in the build container).

usage: python scripts/update_profiles.py <tag>
Reads gpurun_out/{bench.log,bench_ref.log,launches.csv,prof_den.ncu-rep,prof_num.ncu-rep,host.txt}
and writes profiles/<tag>_* plus profiles/ncu_summary.json (used by bench.py's roofline.traffic).
"""
import csv, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return dict(zip(r[0], r[2])), dict(zip(r[0], r[1]))


def to_bytes(v, unit):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main(tag):
    os.makedirs(P, exist_ok=True)
    lines = []
    for f in ("bench.log", "bench_ref.log"):
        p = os.path.join(G, f)
        if os.path.exists(p):
            lines += [l for l in open(p) if l.startswith("{")]
    open(os.path.join(P, f"{tag}_bench.jsonl"), "w").writelines(lines)
    # every config of gpu_final.sh (ours + reference arm), one line each
    cfg = []
    for c in ("wsj_mono", "toy", "hmm", "wsj_biphone", "large", "sweep", "sweep128"):
        for f in ((f"bench_{c}.log", f"bench_ref_{c}.log") if c != "wsj_mono" else
                  ("bench.log", "bench_ref.log")):
            p = os.path.join(G, f)
            if os.path.exists(p):
                cfg += [l for l in open(p) if l.startswith("{")]
    if cfg:
        open(os.path.join(P, f"{tag}_configs.jsonl"), "w").writelines(cfg)
    for f, keep in (("pytest_gpu.log", 12), ("smoke.log", 20), ("sanitizers.log", 20)):
        p = os.path.join(G, f)
        if os.path.exists(p):
            tail = open(p).read().splitlines()[-keep:]
            open(os.path.join(P, f"{tag}_{f}"), "w").write("\n".join(tail) + "\n")
    if os.path.exists(os.path.join(G, "host.txt")):
        open(os.path.join(P, f"{tag}_host.txt"), "w").write(open(os.path.join(G, "host.txt")).read())
    lc = os.path.join(G, "launches.csv")
    if os.path.exists(lc):
        rows = list(csv.reader(open(lc)))
        start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        h = rows[start]
        kn, mv, iid = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
        with open(os.path.join(P, f"{tag}_launches.csv"), "w") as f:
            w = csv.writer(f)
            w.writerow(["id", "kernel", "gpu__time_duration.sum_ns"])
            for r in rows[start + 1:]:
                w.writerow([r[iid], r[kn][:110], r[mv]])
    summ = {"round": tag, "workload": "wsj_mono",
            "source": "ncu --set full --clock-control none; bench.py --profile (wsj_mono, seed 0)"}
    txt = []
    for name in ("den", "num", "chain", "ss", "hmm"):
        rep = os.path.join(G, f"prof_{name}.ncu-rep")
        if not os.path.exists(rep):
            continue
        v, u = raw(rep)
        summ[f"{name}_dram_bytes_per_launch"] = (to_bytes(v["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
                                                 + to_bytes(v["dram__bytes_write.sum"], u["dram__bytes_write.sum"]))
        summ[f"{name}_gpu_time_ms"] = to_bytes(v["gpu__time_duration.sum"], "byte") / (
            1e3 if u["gpu__time_duration.sum"] == "us" else 1)
        txt.append(subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep],
                                  capture_output=True, text=True).stdout)
        txt.append(subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_lines.py"), rep, "30"],
                                  capture_output=True, text=True).stdout)
        txt.append(subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_lines_src.py"), rep,
                                   "30"], capture_output=True, text=True).stdout)
    open(os.path.join(P, f"{tag}_ncu_full_summary.txt"), "w").write("\n".join(txt))
    json.dump(summ, open(os.path.join(P, "ncu_summary.json"), "w"), indent=1)
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
