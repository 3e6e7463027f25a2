"""Build the sm_100a C-ABI library ``libtpde_b200.so`` in-tree with nvcc.

The library is plain CUDA C++ (no torch types), so it is compiled directly
with nvcc rather than through torch's extension machinery.  Output:
``paper_1803_10270_b200/libtpde_b200.so`` (git-ignored, travels to the GPU box
with the gpurun snapshot).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libtpde_b200.so"
INCLUDE = PKG.parent / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS_OBJ = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
             "--expt-relaxed-constexpr", "-Xptxas", "-v"]
if os.environ.get("TPDE_PROBES") == "1":   # clock64 phase probes of the fused ALS kernels (tools/als_phases.py ...)
    FLAGS_OBJ.append("-DTP_ALS_PROBES=1")
OBJ = PKG.parent / "build"


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(CSRC.glob("*.cu"))


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(sources()) + list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    return any(p.stat().st_mtime > t for p in deps)


def _obj(src: Path) -> Path:
    return OBJ / (src.stem + ".o")


def _compile(src: Path):
    """One translation unit -> build/<name>.o (rebuilt when the .cu or any header is newer)."""
    obj = _obj(src)
    hdrs = list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    if obj.exists() and all(p.stat().st_mtime <= obj.stat().st_mtime for p in [src, *hdrs]):
        return obj, None
    cmd = [nvcc(), *ARCH, *FLAGS_OBJ, "-I", str(INCLUDE), "-c", "-o", str(obj) + ".tmp", str(src)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode == 0:
        os.replace(str(obj) + ".tmp", obj)
    return obj, res


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every csrc/*.cu for sm_100a (one nvcc per translation unit, in
    parallel) and link libtpde_b200.so in-tree."""
    if not force and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    OBJ.mkdir(exist_ok=True)
    srcs = sources()
    if force:
        for s_ in srcs:
            _obj(s_).unlink(missing_ok=True)
    with ThreadPoolExecutor(max(1, min(len(srcs), os.cpu_count() or 1))) as pool:
        results = list(pool.map(_compile, srcs))
    log = PKG / "build.log"
    text = []
    for src, (obj, res) in zip(srcs, results):
        if res is not None:
            text.append(" ".join(res.args) + "\n" + res.stdout + res.stderr)
            if res.returncode != 0:
                log.write_text("\n".join(text))
                sys.stderr.write(res.stderr[-8000:])
                raise RuntimeError(f"nvcc failed on {src.name} (see {log})")
    cmd = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", str(LIB) + ".tmp",
           *[str(o) for o, _ in results]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    text.append(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    log.write_text("\n".join(text))
    if res.returncode != 0:
        sys.stderr.write(res.stderr[-8000:])
        raise RuntimeError(f"link failed (see {log})")
    os.replace(str(LIB) + ".tmp", LIB)
    if verbose:
        print("\n".join(text))
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
