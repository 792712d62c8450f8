"""Summarise an ncu report (raw page) into a compact per-kernel table: time, DRAM bytes, issue
activity, occupancy, L2 / shared-memory pipe throughput, L2 atomic sectors and the top stall reasons.  Usage: python scripts/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("time_us", "gpu__time_duration.sum", 1e-3),
    ("dram_rd_MB", "dram__bytes_read.sum", None),
    ("dram_wr_MB", "dram__bytes_write.sum", None),
    ("dram_%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("issue_%", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("warps_%", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("inst_M", "smsp__inst_executed.sum", 1e-6),
    ("lanes/inst", "smsp__thread_inst_executed_per_inst_executed.ratio", 1),
    ("fma_%", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("smem_conf", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
    ("L2_MB", "lts__t_bytes.sum", None),
    ("L2_%", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("smem_%", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 1),
    ("red_sectors_M", "lts__t_sectors_srcunit_tex_op_red.sum", 1e-6),
    ("atom_sectors_M", "lts__t_sectors_srcunit_tex_op_atom.sum", 1e-6),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
    for d in data:
        name = d[hdr.index("Kernel Name")].split("(")[0]
        vals = []
        for lab, key, sc in KEYS:
            if key not in hdr:
                continue
            v = d[hdr.index(key)]
            try:
                f = float(v.replace(",", ""))
            except ValueError:
                vals.append(f"{lab}=?")
                continue
            u = units[hdr.index(key)]
            if sc is None:  # bytes -> MB
                mult = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
                f *= mult
            else:
                if key == "gpu__time_duration.sum":
                    f = f * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(u, 1e-3)
                else:
                    f *= sc
            vals.append(f"{lab}={f:.3g}")
        st = []
        for h in stall:
            try:
                st.append((float(d[hdr.index(h)]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
        st.sort(reverse=True)
        print(f"{name}: " + " ".join(vals))
        print("    stalls/issue: " + ", ".join(f"{n}={v:.2f}" for v, n in st[:6]))


if __name__ == "__main__":
    main(sys.argv[1])
