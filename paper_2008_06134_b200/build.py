"""Build the in-tree CUDA library ``_sbrc.so`` for sm_100a with nvcc.

    python paper_2008_06134_b200/build.py

No torch headers are involved: the library exposes the plain C ABI of
include/sbrc.h and is loaded with ctypes.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
#: translation units: the C ABI, and march_inst.cu once per (shading mode, voxel type) with the
#: defines that select it (K2 instantiations compile in parallel; the cone ones are the long pole)
UNITS = [("sbrc.cu", ())] + [("march_inst.cu", (f"SBRC_INST_SHADE={sh}", f"SBRC_INST_VT={vt}"))
                             for sh in (5, 3, 2, 1, 4, 0) for vt in (0, 1, 2)]
SOURCES = ["sbrc.cu", "march_inst.cu"]
SRC = os.path.join(CSRC, "sbrc.cu")
OUT = os.path.join(HERE, "_sbrc.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3", "-shared",
    "-I", os.path.join(ROOT, "include"),
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def build(verbose: bool = False, force: bool = False, out: str = OUT, defines=(), jobs: int | None = None,
          unit_defines=None, obj_cache: str | None = None) -> str:
    """Compile every translation unit (in parallel) and link ``out``; ``defines``
    (e.g. ["SBRC_WIDE_MAX_PIXELS=0"]) and ``out`` build experiment variants.
    ``unit_defines`` ({"sbrc.cu": [...]}) adds defines to one source only, and
    ``obj_cache`` (a directory) keeps the objects, reusing each one that is
    newer than the sources for the same defines — so a K1-only variant
    recompiles sbrc.cu alone."""
    import concurrent.futures as cf
    import hashlib
    import tempfile
    srcs = [os.path.join(CSRC, f) for f in SOURCES]
    deps = srcs + [os.path.join(CSRC, "sbrc_common.cuh"), os.path.join(ROOT, "include", "sbrc.h")]
    if not force and os.path.exists(out) and all(os.path.getmtime(out) >= os.path.getmtime(d) for d in deps):
        return out
    tmp = obj_cache or tempfile.mkdtemp(prefix="sbrc_build_")
    os.makedirs(tmp, exist_ok=True)
    newest = max(os.path.getmtime(d) for d in deps)
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]
    extra = [f"-D{d}" for d in defines] + (["-Xptxas", "-v"] if verbose else [])

    def compile_one(unit):
        name, defs = unit
        src = os.path.join(CSRC, name)
        cmd = [nvcc(), *compile_flags, *[f"-D{d}" for d in defs], *extra,
               *[f"-D{d}" for d in (unit_defines or {}).get(name, ())]]
        key = hashlib.sha1(" ".join(cmd).encode()).hexdigest()[:12]
        obj = os.path.join(tmp, "_".join([name] + [d.split("=")[1] for d in defs] + [key]) + ".o")
        if obj_cache and not verbose and os.path.exists(obj) and os.path.getmtime(obj) >= newest:
            return src, obj, subprocess.CompletedProcess(cmd, 0, "", "")
        res = subprocess.run([*cmd, "-c", "-o", obj, src], capture_output=True, text=True)
        return src, obj, res

    with cf.ThreadPoolExecutor(max_workers=jobs or min(len(UNITS), os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, UNITS))
    for src, obj, res in results:
        if verbose:
            sys.stderr.write(res.stderr)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {os.path.basename(src)} ({res.returncode}):\n{res.stderr}")
    link = subprocess.run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out + ".tmp",
                           *[obj for _, obj, _ in results]], capture_output=True, text=True)
    if link.returncode != 0:
        raise RuntimeError(f"nvcc link failed ({link.returncode}):\n{link.stderr}")
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(verbose="-v" in sys.argv, force=True, out=outs[0] if outs else OUT, defines=defs))
