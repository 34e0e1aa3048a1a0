"""Copy the reference's committed test fixture data (proj/tests/fixtures/gaussian,
used by proj/tests/test_io_cli.cpp:276-300) into tests/golden/ so the CSV
reader/writer can be pinned against real reference-written files on machines
without /root/reference.  Data files only (no source).  Run once here:

    python tools/make_golden.py
"""
import os
import shutil
import sys

SRC = "/root/reference/proj/tests/fixtures/gaussian"
DST = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "gaussian_fixture")

if __name__ == "__main__":
    if not os.path.isdir(SRC):
        sys.exit("reference fixtures not present: " + SRC)
    os.makedirs(DST, exist_ok=True)
    for name in ("X1.csv", "X2.csv", "expected.json"):
        shutil.copyfile(os.path.join(SRC, name), os.path.join(DST, name))
        print("copied", name)
