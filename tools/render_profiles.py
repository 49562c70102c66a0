"""Render profiles/ from a make_profiles.sh run (gpurun_out/): launch list
of one step, ncu --set full summary, per-kernel DRAM traffic (traffic.json,
read by bench.py), SASS listings of the hot kernels.
    python tools/render_profiles.py ROUND   (e.g. r01)"""
import csv
import io
import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"

GROUPS = {  # bench.py kernel-table names
    "k_keys": "bucket_keys(K1a)", "k_radix_scatter": "bucket_scatter(K1c)",
    "k_grid_items": "grid(K2)", "k_fft_rows": "fft_rows(K3a)",
    "k_fft_cols": "fft_cols_stack(K3b+K4)",
}


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
    PROF.mkdir(exist_ok=True)
    subprocess.run([sys.executable, str(ROOT / "tools/launch_summary.py"),
                    str(OUT / "launches_raw.csv"), str(PROF / f"launches_{rnd}.csv")], check=True,
                   capture_output=True)
    if (OUT / "launches_cfg3_raw.csv").exists():
        subprocess.run([sys.executable, str(ROOT / "tools/launch_summary.py"),
                        str(OUT / "launches_cfg3_raw.csv"), str(PROF / f"launches_cfg3_{rnd}.csv")],
                       check=True, capture_output=True)
    rep = OUT / "full.ncu-rep"
    txt = subprocess.run([sys.executable, str(ROOT / "tools/ncu_summary.py"), str(rep)],
                         capture_output=True, text=True).stdout
    (PROF / f"ncu_{rnd}.txt").write_text(txt)
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    ki, rd, wr = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    traffic = {}
    for r in rows[2:]:
        name = r[ki]
        for k, g in GROUPS.items():
            if re.search(k + r"\b", name):
                b = (float(r[rd].replace(",", "")) * scale.get(units[rd], 1) +
                     float(r[wr].replace(",", "")) * scale.get(units[wr], 1))
                traffic.setdefault(g, int(b))   # first launch of the kind
    (PROF / "traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
    print(json.dumps(traffic, indent=1))
    sass_listings()


# hot kernels whose SASS is kept: (file stem, regex on the mangled name)
SASS = (("k_grid_items_0_3", r"k_grid_itemsILi0ELi3E"), ("k_fft_rows_11", r"k_fft_rowsILi11ELi0E7double2"),
        ("k_fft_cols_11", r"k_fft_colsILi11ELi0E7double2"), ("k_fft_cols_11_fp32", r"k_fft_colsILi11ELi0E6float2"),
        ("k_radix_scatter_8", r"k_radix_scatterILi8ELb0E"), ("k_keys", r"k_keysILb1E"),
        ("k_prepare", r"k_prepareEPK"), ("k_push", r"k_push[^4]"), ("k_image_finish", r"k_image_finish"),
        ("k_route_pack", r"k_route_pack"))


def sass_listings():
    """cuobjdump -sass of the in-tree libwsb.so, one file per hot kernel,
    instruction encodings stripped."""
    so = ROOT / "paper_2504_00959_b200" / "libwsb.so"
    dump = subprocess.run(["cuobjdump", "-sass", str(so)], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", dump)
    out = PROF / "sass"
    out.mkdir(exist_ok=True)
    for stem, pat in SASS:
        for f in funcs[1:]:
            name = f.split("\n", 1)[0]
            if re.search(pat, name):
                body = re.sub(r"\s*/\* 0x[0-9a-f]{16} \*/", "", f)
                body = "\n".join(l for l in body.splitlines() if l.strip())
                (out / f"{stem}.sass").write_text("Function : " + body + "\n")
                break


if __name__ == "__main__":
    main()
