"""Hot CUDA source lines of one kernel in an ncu report (needs -lineinfo):
instructions executed and stall samples per source line (SASS attributed).
    python tools/src_hot.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep, pat = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + pat,
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    cur_file = ""
    agg = {}
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or not r[0].isdigit():
            continue
        try:
            ex = int(r[hdr.index("Instructions Executed")] or 0)
            st = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        key = (cur_file, int(r[0]))
        e = agg.setdefault(key, [0, 0, r[1].strip()[:90]])
        e[0] += ex
        e[1] += st
    tot = sum(v[0] for v in agg.values()) or 1
    tst = sum(v[1] for v in agg.values()) or 1
    for (f, ln), (ex, st, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{ex / tot:6.1%} {st / tst:6.1%}  {f}:{ln}  {src}")


if __name__ == "__main__":
    main()
