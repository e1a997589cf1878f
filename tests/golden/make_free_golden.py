"""Generate tests/golden/free_api_ref.bin.gz (and free_api_ref_s<seed>.bin.gz
for the seeded random variants): the output of
tests/native/free_api_test.cpp compiled against the REFERENCE headers and
linked with the reference objects oracle/Makefile builds from
/root/reference/proj (run in the build container, where the reference is
present).  The GPU test runs the same program built against include/ and
libswflood_b200.so and compares the bytes (tests/test_dropin_cpp.py).

    python tests/golden/make_free_golden.py
"""
import gzip
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_INC = "/root/reference/proj/include"
OUT = os.path.join(HERE, "free_api_ref.bin.gz")
REF_OBJS = ["grid", "block", "sources", "forcing", "riemann", "stepper", "ref_shim"]


def build_ref_exe(exe):
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True,
                   stdout=subprocess.DEVNULL)
    objs = [os.path.join(ROOT, "oracle", "_ref", o + ".o") for o in REF_OBJS]
    cmd = ["/usr/bin/g++", "-std=c++20", "-O3", "-ffp-contract=off", "-fopenmp",
           "-I", os.path.join(ROOT, "oracle", "_ref", "include"), "-I", REF_INC,
           os.path.join(ROOT, "tests", "native", "free_api_test.cpp")] + objs + ["-o", exe]
    subprocess.run(cmd, check=True)
    return exe


SEEDS = range(1, 9)  # the seeded random variants (free_api_test.cpp argv[2])


def seeded_path(seed):
    return os.path.join(HERE, f"free_api_ref_s{seed}.bin.gz")


def reference_output(seed=0):
    with tempfile.TemporaryDirectory() as d:
        exe = build_ref_exe(os.path.join(d, "free_ref"))
        out = os.path.join(d, "free_ref.bin")
        subprocess.run([exe, out] + ([str(seed)] if seed else []), check=True,
                       stdout=subprocess.DEVNULL)
        with open(out, "rb") as f:
            return f.read()


def main():
    for seed in [0] + list(SEEDS):
        data = reference_output(seed)
        path = OUT if seed == 0 else seeded_path(seed)
        with gzip.open(path, "wb", compresslevel=9) as f:
            f.write(data)
        print(f"{path}: {len(data)} bytes")


if __name__ == "__main__":
    sys.exit(main())
