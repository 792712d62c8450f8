"""The boundary is a C ABI: a plain C program (gcc, no C++ / CUDA / torch headers) includes
include/rtgs.h, links librtgs.so and exercises the host-side calls (no GPU needed)."""
import os
import subprocess

import pytest

from paper_2404_19706_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_plain_c_client(tmp_path):
    B.build()
    lib_dir = os.path.dirname(B.LIB)
    exe = str(tmp_path / "abi_smoke")
    cmd = ["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "c", "abi_smoke.c"), "-L", lib_dir, "-lrtgs", f"-Wl,-rpath,{lib_dir}",
           "-o", exe]
    if subprocess.run(["which", "gcc"], capture_output=True).returncode != 0:
        pytest.skip("gcc not available")
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c abi ok" in r.stdout
