"""Per-CUDA-line instruction / stall shares of one ncu report (source page, cuda,sass)."""
import csv, subprocess, sys, io

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
f = "?"
agg = []
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0].isdigit():
        try:
            st, ex = int(r[4]), int(r[7])
        except ValueError:
            continue
        agg.append((f, int(r[0]), r[1].strip()[:90], st, ex))
tst = sum(a[3] for a in agg) or 1
tex = sum(a[4] for a in agg) or 1
print(f"total warp insts {tex}, stall samples {tst}")
for a in sorted(agg, key=lambda a: -(a[3] / tst + a[4] / tex))[:n]:
    print(f"{a[0]}:{a[1]:<5} inst {100*a[4]/tex:5.1f}%  stall {100*a[3]/tst:5.1f}%  {a[2]}")
