"""Executed instructions and stall samples of one kernel in an ncu report, aggregated per CUDA source
line (needs -lineinfo and --import-source on).  python scripts/ncu_lines.py report kernel_regex [top]"""
import csv
import io
import subprocess
import sys


def main(path, kernel, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name", f"regex:{kernel}", "--launch-skip", sys.argv[4] if len(sys.argv) > 4 else "0",
                          "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    f = lambda v: float(v) if v.replace(".", "", 1).isdigit() else 0.0
    rows, fname = [], ""
    for r in csv.reader(io.StringIO(out)):
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif len(r) > 8 and r[0] not in ("", "Line No"):  # a source line with its aggregated metrics
            rows.append((fname, r[0], r[1], f(r[7]), f(r[4])))
    ti = sum(x[3] for x in rows)
    ts = sum(x[4] for x in rows)
    print(f"instructions {ti:.4g}  samples {ts:.4g}")
    rows.sort(key=lambda x: -x[3])
    for fn, ln, src, i, s in rows[:top]:
        print(f"{fn}:{ln:<5} {100 * i / ti:5.1f}%i {100 * s / max(ts, 1):5.1f}%s  {src.strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
