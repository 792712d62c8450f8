"""Hottest SASS instructions of one kernel in an ncu report (by warp-stall samples and executed
instructions).  Usage: python scripts/ncu_hot.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys


def main(path, kernel, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name", f"regex:{kernel}",
                          "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    f = lambda v: float(v) if v.replace(".", "", 1).isdigit() else 0.0
    tot_s = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in data)
    tot_i = sum(f(d["Instructions Executed"]) for d in data)
    print(f"instructions {tot_i:.3g}  stall samples {tot_s:.3g}")
    data.sort(key=lambda d: -f(d["Warp Stall Sampling (All Samples)"]))
    for d in data[:top]:
        s = f(d["Warp Stall Sampling (All Samples)"])
        i = f(d["Instructions Executed"])
        print(f"{d['Address']:>6} {100 * s / tot_s:5.1f}%s {100 * i / tot_i:5.1f}%i  {d['Source'][:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
