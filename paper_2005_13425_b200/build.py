"""Build libsem.so in-tree for sm_100a (``python -m paper_2005_13425_b200.build``).

The library is plain nvcc output (static cudart, no torch symbols) so it can
be loaded by ctypes from any host language; see include/sem.h.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsem.so")
# ax_inst.cu is compiled once per n group (-DSEM_AX_GROUP=k) so the unrolled
# per-n Ax instantiations build in parallel.
AX_GROUPS = 8
SOURCES = ["common.cu", "ax.cu", "ax_variants.cu", "assembly.cu", "cg.cu", "fields.cu", "host.cu", "slab.cu", "probe.cu"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    cand = os.path.join(cuda, "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "sem.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile_flags(verbose: bool = False) -> list:
    flags = [f for f in NVCC_FLAGS if f != "-shared"]
    # tuning experiments: extra -D definitions (e.g. SEM_NVCC_DEFS="SEM_UPD_MINB=8")
    flags += [f"-D{d}" for d in os.environ.get("SEM_NVCC_DEFS", "").split()]
    if verbose:
        flags += ["-Xptxas", "-v"]
    return flags


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every translation unit concurrently (one nvcc per .cu), then
    link the shared library.  Rebuilt when a source is newer than the library
    or the -D set (SEM_NVCC_DEFS) differs from the one it was built with."""
    compile_flags = _compile_flags(verbose)
    flag_file = OUT + ".flags"
    built_with = open(flag_file).read() if os.path.exists(flag_file) else None
    if not force and not _stale() and built_with == " ".join(compile_flags):
        return OUT
    # objects are cached per flag set outside the tree (SEM_OBJ_CACHE): a unit
    # is recompiled when its .cu, any header or the flags changed
    cache = os.environ.get("SEM_OBJ_CACHE")
    if cache and not force:
        import hashlib
        key = hashlib.sha1(" ".join(compile_flags).encode()).hexdigest()[:12]
        objdir = os.path.join(cache, key)
        os.makedirs(objdir, exist_ok=True)
    else:
        objdir = tempfile.mkdtemp(prefix="libsem_obj_")
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    headers.append(os.path.join(HERE, "..", "include", "sem.h"))
    t_hdr = max(os.path.getmtime(h) for h in headers if os.path.exists(h))
    units = [(src, src.replace(".cu", ".o"), []) for src in SOURCES]
    units += [("ax_inst.cu", f"ax_inst{k}.o", [f"-DSEM_AX_GROUP={k}"]) for k in range(AX_GROUPS)]
    units.sort(key=lambda u: u[0] != "ax_inst.cu")  # longest jobs first
    procs, objs = [], []
    for src, objname, extra in units:
        obj = os.path.join(objdir, objname)
        objs.append(obj)
        if os.path.exists(obj) and os.path.getmtime(obj) > max(
                t_hdr, os.path.getmtime(os.path.join(CSRC, src))):
            continue
        cmd = [nvcc(), *compile_flags, *extra, "-c", "-o", obj, os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((src, subprocess.Popen(cmd)))
    failed = [src for src, p in procs if p.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, f"nvcc ({', '.join(failed)})")
    link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
            "-o", OUT + ".tmp", *objs]
    subprocess.run(link, check=True)
    os.replace(OUT + ".tmp", OUT)
    with open(flag_file, "w") as fh:
        fh.write(" ".join(compile_flags))
    if not (cache and not force):
        shutil.rmtree(objdir, ignore_errors=True)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
