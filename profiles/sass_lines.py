"""Aggregate an ncu source page (SASS, CSV) by CUDA source line.

    ncu -i rep --page source --csv --print-source sass > sass.csv
    nvdisasm -g -c <cubin> > all.dis        (cuobjdump -xelf all <obj> for the cubin)
    python profiles/sass_lines.py sass.csv all.dis <mangled kernel name> [top]

Prints per file:line the warp-stall samples, executed warp instructions and
the dominant stall reasons (line info of the outermost inlined frame)."""
import csv
import re
import sys
from collections import defaultdict


def line_map(dis, fn):
    out, cur, on = {}, None, False
    for ln in open(dis):
        if ln.startswith("//---------------------"):
            on = (".text." + fn + " ") in ln
            continue
        if not on:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
            continue
        m = re.match(r"\s+/\*([0-9a-f]+)\*/", ln)
        if m:
            out[int(m.group(1), 16)] = cur
    return out


def main():
    csvf, dis, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    lm = line_map(dis, fn)
    rows = list(csv.reader(open(csvf)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    base = None
    agg = defaultdict(lambda: defaultdict(float))
    tot = defaultdict(float)
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        try:
            addr = int(r[ix["Address"]], 16)
        except ValueError:
            continue
        if base is None:  # the page lists absolute addresses, kernel entry first
            base = addr
        addr -= base
        key = lm.get(addr, "?")
        a = agg[key]
        for h in ["Warp Stall Sampling (All Samples)", "Instructions Executed"] + stalls:
            v = float(r[ix[h]] or 0)
            a[h] += v
            tot[h] += v
    S, I = "Warp Stall Sampling (All Samples)", "Instructions Executed"
    print(f"total samples {tot[S]:.0f}, warp instructions {tot[I]:.0f}")
    for key, a in sorted(agg.items(), key=lambda kv: -kv[1][S])[:top]:
        st = sorted(((a[h], h[6:]) for h in stalls), reverse=True)[:3]
        sts = ", ".join(f"{n} {v / max(a[S], 1):.0%}" for v, n in st if v > 0)
        print(f"{key:28s} samples {a[S] / tot[S]:6.1%}  instr {a[I] / tot[I]:6.1%}  {sts}")


if __name__ == "__main__":
    main()
