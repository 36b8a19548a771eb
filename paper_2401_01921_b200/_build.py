"""Build libtnb.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

``python -m paper_2401_01921_b200._build`` or ``__graft_entry__.build()``.
The .so lands next to this file so it travels with the repo snapshot.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtnb.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith((".cu", ".cpp")))


def headers():
    inc = os.path.join(os.path.dirname(HERE), "include")
    out = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    out += [os.path.join(inc, f) for f in os.listdir(inc) if f.endswith(".h")]
    return out


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in sources() + headers())


def build(force=False, verbose=False, defines=(), out=None):
    """Compile every csrc/ source for sm_100a and link libtnb.so. `defines` / `out` build
    a variant (e.g. ``-DTNB_X=1`` into build/variant.so) for A/B measurements."""
    lib = out or LIB
    if not force and not defines and out is None and up_to_date():
        return LIB
    objdir = os.path.join(HERE, "build", os.path.splitext(os.path.basename(lib))[0]) if out else os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", *defines, "-Xcompiler", "-fPIC,-O3",
               "-Xptxas", "-v" if verbose else "-O3", "-c", src, "-o", obj]
        if src.endswith(".cpp"):
            cmd = [NVCC, "-x", "cu", *cmd[1:]]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(out.decode())
        if p.returncode != 0:
            failed = True
            sys.stderr.write(f"[tnb build] FAILED: {src}\n")
    if failed:
        raise RuntimeError("libtnb build failed")
    tmp = lib + ".tmp"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    defs = [a for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[len("--out="):] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs, out=outs[0] if outs else None))
