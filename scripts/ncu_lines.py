"""Per-CUDA-source-line instruction / stall attribution from an ncu report
(`--page source --print-source=cuda,sass`), run in the build container."""
import csv, io, subprocess, sys
from collections import defaultdict

def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    fpath = None; hdr = None
    agg = defaultdict(lambda: [0, 0, 0, ""])
    cur_line = None
    for r in csv.reader(io.StringIO(out)):
        if not r: continue
        if r[0] == "File Path": fpath = r[1].split("/")[-1]; continue
        if r[0] == "Line No": hdr = r; continue
        if hdr is None or r[0] in ("Function Name",): continue
        if r[0].isdigit():
            cur_line = (fpath, int(r[0]), r[1][:90])
            ie = hdr.index("Instructions Executed"); st = hdr.index("Warp Stall Sampling (All Samples)")
            wf = hdr.index("L1 Wavefronts Shared")
            def num(x):
                try: return float(x)
                except: return 0.0
            a = agg[cur_line]
            a[0] += num(r[ie]); a[1] += num(r[st]); a[2] += num(r[wf])
    ti = sum(v[0] for v in agg.values()) or 1; ts = sum(v[1] for v in agg.values()) or 1
    tw = sum(v[2] for v in agg.values()) or 1
    print(f"total warp-inst {ti:.3e}  stall samples {ts:.0f}  smem wavefronts {tw:.3e}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{k[0]}:{k[1]:4d} inst {v[0]/ti*100:5.1f}% stall {v[1]/ts*100:5.1f}% wf {v[2]/tw*100:5.1f}% | {k[2]}")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
