"""Build libdrb200.so in-tree with nvcc for sm_100a (no JIT cache, travels with gpurun).

    python -m paper_2509_10466_b200.build            # incremental
    python -m paper_2509_10466_b200.build --force
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_build"
LIB = OUT_DIR / "libdrb200.so"
SOURCES = ["engine.cu", "mask_kernels.cu", "token_tc.cu", "attention_tc.cu",
           "conv_tc.cu", "v2p_tc.cu", "dec_fused.cu", "frame_ops.cu"]
HEADERS = ["common.cuh", "kernels.h", "tc.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills"]


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src] + [CSRC / h for h in HEADERS] + [PKG.parent / "include" / "dr_b200.h"]
    return any(d.stat().st_mtime > obj.stat().st_mtime for d in deps)


def build(force: bool = False, verbose: bool = False, trace: bool = False,
          variant: str = "", defines=()) -> Path:
    """trace=True builds a separate diagnostic library (_build_trace/, -DDR_TRACE: per-CTA
    timer stamps, scripts/*_trace.py) -- never the product.  variant/defines build an A/B
    experiment library into _build_<variant>/ (select it with DR_B200_LIB)."""
    out_dir = PKG / "_build_trace" if trace else (PKG / f"_build_{variant}" if variant else OUT_DIR)
    lib_path = out_dir / LIB.name
    flags = FLAGS + (["-DDR_TRACE"] if trace else []) + list(defines)
    out_dir.mkdir(exist_ok=True)
    objs = []
    for name in SOURCES:
        src = CSRC / name
        obj = out_dir / (name + ".o")
        objs.append(obj)
        if force or _stale(obj, src):
            cmd = [NVCC, *ARCH, *flags, "-c", str(src), "-o", str(obj)]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            print("[build]", " ".join(cmd[-3:]), flush=True)
            subprocess.run(cmd, check=True)
    if force or not lib_path.exists() or any(o.stat().st_mtime > lib_path.stat().st_mtime
                                             for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(lib_path), *map(str, objs), "-lcudart_static",
               "-lrt", "-ldl", "-lpthread"]
        print("[build] link", lib_path.relative_to(PKG), flush=True)
        subprocess.run(cmd, check=True)
    return lib_path


if __name__ == "__main__":
    defs = [a for a in sys.argv[1:] if a.startswith("-D")]
    var = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--variant=")), "")
    build(force="--force" in sys.argv, verbose="-v" in sys.argv, trace="--trace" in sys.argv,
          variant=var, defines=defs)
