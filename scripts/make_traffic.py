"""profiles/traffic.json from the measurement pass's ncu --set full captures: per bench config, DRAM
bytes (read + write) per launch of the kernels the bench line cites, and the FULL render's executed
warp instructions.  python scripts/make_traffic.py gpurun_out/r2m_prof.ncu-rep gpurun_out/r2m_prof_c4.ncu-rep"""
import csv
import io
import json
import subprocess
import sys

WANT = {  # bench key -> kernel name prefix in the report (first launch that matches)
    "C3": {"k_render_fwd<FULL>": "void k_render_fwd<0, 0, 0, 1>", "k_project": "void k_project<16, 0>",
           "k_render_bwd": "k_render_bwd", "k_project_bwd<ADAM>": "void k_project_bwd<16, 1>"},
    "C4": {"k_render_fwd<FULL>": "void k_render_fwd<0, 0, 0, 1>", "k_project": "void k_project<16, 0>"},
}


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    units = dict(zip(r[0], r[1]))  # the second row holds each column's unit
    res = []
    for v in r[2:]:
        d = dict(zip(r[0], v))
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            d[k] = float(d[k].replace(",", "")) * SCALE.get(units.get(k, "byte"), 1)
        res.append(d)
    return res


def main(c3, c4):
    res = {"_source": "scripts/make_traffic.py: ncu --set full --clock-control none captures of the final round-2 "
                      "build (scripts/r2_measure.sh); dram__bytes_read.sum + dram__bytes_write.sum per launch; "
                      "*_warp_inst = smsp__inst_executed.sum of the same capture; k_render_fwd<FULL> = the "
                      "production span variant k_render_fwd<0, 0, 0, 1>; keyed by bench config"}
    for cfg, path in (("C3", c3), ("C4", c4)):
        d, rs = {}, rows(path)
        for key, name in WANT[cfg].items():
            for r in rs:
                if r["Kernel Name"].startswith(name):
                    d[key] = int(r["dram__bytes_read.sum"] + r["dram__bytes_write.sum"])
                    if key == "k_render_fwd<FULL>":
                        d[key + "_warp_inst"] = int(float(r["smsp__inst_executed.sum"].replace(",", "")))
                    break
        res[cfg] = d
    json.dump(res, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
