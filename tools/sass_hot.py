"""Hot SASS of one kernel in an ncu report: instructions executed and stall
samples per instruction, plus totals per contiguous block between branches.
    python tools/sass_hot.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep, pat = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + pat,
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    iex = hdr.index("Instructions Executed")
    ist = hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        try:
            data.append((r[ia], r[isrc].strip(), int(r[iex] or 0), int(r[ist] or 0)))
        except ValueError:
            pass
    tot_ex = sum(d[2] for d in data)
    tot_st = sum(d[3] for d in data)
    print(f"instructions {tot_ex}  stall samples {tot_st}")
    # blocks: runs of instructions with equal execution count
    blocks = []
    cur = None
    for i, d in enumerate(data):
        if cur is None or d[2] != cur[2]:
            cur = [i, i, d[2], 0, 0]
            blocks.append(cur)
        cur[1] = i
        cur[3] += d[2]
        cur[4] += d[3]
    blocks.sort(key=lambda b: -b[3])
    for b in blocks[:top]:
        i0, i1 = b[0], b[1]
        ops = {}
        for d in data[i0:i1 + 1]:
            op = d[1].split()[0] if d[1] else "?"
            if op.startswith("@"):
                op = d[1].split()[1]
            op = op.split(".")[0]
            ops[op] = ops.get(op, 0) + 1
        opstr = " ".join(f"{k}x{v}" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:8])
        print(f"{data[i0][0]}-{data[i1][0]} n={i1 - i0 + 1:3d} exec/inst={b[2]:>10d} "
              f"share={b[3] / tot_ex:5.1%} stall={b[4] / max(tot_st, 1):5.1%}  {opstr}")


if __name__ == "__main__":
    main()
