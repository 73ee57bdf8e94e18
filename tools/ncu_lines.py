"""Per-source-line stall samples and instructions of one kernel in an ncu
report (ncu -i REP --page source --csv --print-source cuda,sass): the top
lines by warp-stall samples, with the file they belong to."""
import csv
import subprocess
import sys


def main(rep, kernel, top=40):
    out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kernel}", "--page", "source", "--csv",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    fname, hdr, agg = None, None, {}
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0]:
            continue  # SASS rows carry an empty line number
        try:
            samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            inst = int(r[hdr.index("Instructions Executed")])
        except (ValueError, IndexError):
            continue
        key = (fname, int(r[0]))
        s = agg.setdefault(key, [0, 0, r[1][:90]])
        s[0] += samp
        s[1] += inst
    tot = sum(v[0] for v in agg.values()) or 1
    toti = sum(v[1] for v in agg.values()) or 1
    print(f"total samples {tot}, warp instructions {toti}")
    for (f, ln), (s, i, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100*s/tot:5.1f}% smp {100*i/toti:5.1f}% ins  {f}:{ln:<5} {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
