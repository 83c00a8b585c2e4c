"""Copy the reference's own API tests (pkg/tests: the cgemm /
rgemm / lu / ozaki suites) into tests/ref_suite/_vendored/ -- a git-ignored
directory (reference sources never enter this repo's history) that travels
to the GPU box with the gpurun snapshot.  tests/ref_suite/conftest.py then
runs them against this package through sys.modules["mpclu"] (SURVEY.md §7.2,
VERDICT r1 item 8).  Run here (the reference tree exists only in this
container):  python tools/vendor_ref_suite.py"""
import os
import shutil

SRC = "/root/reference/pkg/tests"
DST = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                   "ref_suite", "_vendored")
# the suites only use the reference conftest's `rng` fixture, which
# tests/ref_suite/conftest.py provides; files are renamed test_ref_* so their
# module names cannot collide with this repo's own tests
FILES = ["test_cgemm.py", "test_rgemm.py", "test_lu.py", "test_ozaki.py"]

if __name__ == "__main__":
    os.makedirs(DST, exist_ok=True)
    for f in FILES:
        shutil.copyfile(os.path.join(SRC, f), os.path.join(DST, f.replace("test_", "test_ref_", 1)))
    print("vendored", len(FILES), "files into", DST)
