"""Per-CUDA-source-line instruction / warp-stall totals from an ncu report
(the `--print-source cuda,sass` source page; needs -lineinfo builds).

    python profiles/cuda_lines.py gpurun_out/x.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def lines(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    f, hdr, res = None, None, []
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if hdr is None or not r[0]:
            continue
        try:
            ie = int(r[hdr["Instructions Executed"]] or 0)
            ss = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        except (ValueError, KeyError, IndexError):
            continue
        res.append((ie, ss, f"{f}:{r[0]}", r[1].strip()[:100]))
    return res


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    res = lines(rep)
    ti = sum(x[0] for x in res) or 1
    ts = sum(x[1] for x in res) or 1
    print(f"warp instructions {ti}, stall samples {ts}")
    for ie, ss, loc, src in sorted(res, reverse=True)[:top]:
        print(f"{100 * ie / ti:6.2f}% inst {100 * ss / ts:6.2f}% samples  {loc:24s} {src}")


if __name__ == "__main__":
    main()
