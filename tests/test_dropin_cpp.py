"""The C++ drop-in (include/swflood/*.hpp + libswflood_b200.so): a program
written against the reference's API compiles here; on the GPU it runs and
matches the C restatement bit for bit."""
import os
import subprocess

import pytest

from conftest import ROOT

EXE = os.path.join(ROOT, "tests", "native", "dropin_test")


def build_exe():
    from paper_1705_00614_b200 import build as b
    b.build()
    from oracle import pyorc
    if not pyorc.available("orc"):
        pyorc.build(ref=False)
    pkg = os.path.join(ROOT, "paper_1705_00614_b200")
    cmd = ["/usr/bin/g++", "-std=c++20", "-O2", "-ffp-contract=off",
           "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "native", "dropin_test.cpp"),
           "-o", EXE, "-L", pkg, "-lswflood_b200", "-lswflood_cuda",
           os.path.join(ROOT, "oracle", "liborc.so"),
           f"-Wl,-rpath,{pkg}", f"-Wl,-rpath,{os.path.join(ROOT, 'oracle')}"]
    subprocess.run(cmd, check=True)
    return EXE


def test_dropin_compiles():
    assert os.path.exists(build_exe())


@pytest.mark.gpu
def test_dropin_runs_bit_exact():
    exe = build_exe()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "dropin ok" in r.stdout


NEST_EXE = os.path.join(ROOT, "tests", "native", "nest_io_test")


def build_nest_exe():
    from paper_1705_00614_b200 import build as b
    b.build()
    pkg = os.path.join(ROOT, "paper_1705_00614_b200")
    cmd = ["/usr/bin/g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "native", "nest_io_test.cpp"), "-o", NEST_EXE, "-L", pkg,
           "-lswflood_b200", "-lswflood_cuda", f"-Wl,-rpath,{pkg}"]
    subprocess.run(cmd, check=True)
    return NEST_EXE


def test_nest_io_program_compiles():
    assert os.path.exists(build_nest_exe())


@pytest.mark.gpu
def test_nest_io_program_runs(tmp_path):
    exe = build_nest_exe()
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "nest_io ok" in r.stdout
