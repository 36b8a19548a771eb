"""Stage the reference (tnkit) and its own test suite under baseline/_ref (git-ignored; it
travels to the GPU box with the repo snapshot, /root/reference does not).

    python integration/prepare_reference_suite.py [/root/reference]

1. ``pip install --no-index --no-build-isolation --no-deps --target baseline/_ref`` of
   pkg/ from a scratch copy under /tmp (the reference tree is read-only; numpy/scipy are
   already in the image, so dependency resolution is skipped with --no-deps);
2. a scratch copy of pkg/tests as baseline/_ref/suite/tests with an empty __init__.py
   (the suite imports ``from tests.conftest import ...``).
Nothing here is committed: the reference's sources stay out of the repository history.
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def main(ref="/root/reference"):
    pkg = os.path.join(ref, "pkg")
    if not os.path.isdir(pkg):
        raise SystemExit(f"{pkg}: reference package not found")
    tmp = tempfile.mkdtemp(prefix="tnkit_ref_")
    try:
        shutil.copytree(pkg, os.path.join(tmp, "pkg"))
        if not os.path.isdir(os.path.join(REF_DIR, "tnkit")):
            subprocess.check_call([sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
                                   "--no-deps", "--find-links", "/opt/wheelhouse", "--target", REF_DIR,
                                   os.path.join(tmp, "pkg")])
        suite = os.path.join(REF_DIR, "suite")
        shutil.rmtree(suite, ignore_errors=True)
        shutil.copytree(os.path.join(tmp, "pkg", "tests"), os.path.join(suite, "tests"))
        open(os.path.join(suite, "tests", "__init__.py"), "a").close()
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    print(REF_DIR)


if __name__ == "__main__":
    main(*sys.argv[1:])
