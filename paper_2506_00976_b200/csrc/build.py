"""Build libgridot_b200.so in-tree with nvcc (sm_100a) and g++.

    python -m paper_2506_00976_b200.csrc.build        # incremental
    python -m paper_2506_00976_b200.csrc.build --force

Object files go to csrc/_obj/; the shared library lands next to this file so
it travels to the GPU box with the repo snapshot (git-ignored).
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
OBJ = os.path.join(HERE, "_obj")
LIB = os.path.join(HERE, "libgridot_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
           "--expt-relaxed-constexpr"] + ARCH
# files whose arithmetic restates the reference's rounding order: no FMA
NO_FMA = {"grid_kernels.cu", "primal.cu", "cbar.cu", "entropic.cu"}
CU = ["grid_kernels.cu", "cbar.cu", "cbar_fast.cu", "cbar_diag.cu", "primal.cu", "ctransform.cu",
      "ctransform_pruned.cu", "entropic.cu", "probes.cu"]
CPP = ["simplex.cpp"]
HEADERS = ["common.cuh", os.path.join("..", "..", "include", "gridot_b200.h")]


def _newer(src_list, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in src_list)


def _run(cmd, log):
    res = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd)}")


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    hdrs = [os.path.join(HERE, h) for h in HEADERS]
    objs, jobs = [], []
    for f in CU:
        src = os.path.join(HERE, f)
        obj = os.path.join(OBJ, f + ".o")
        objs.append(obj)
        if force or _newer([src] + hdrs + [__file__], obj):
            flags = NVFLAGS + (["--fmad=false"] if f in NO_FMA else [])
            jobs.append((f, [NVCC] + flags + ["-c", src, "-o", obj]))
    for f in CPP:
        src = os.path.join(HERE, f)
        obj = os.path.join(OBJ, f + ".o")
        objs.append(obj)
        if force or _newer([src] + hdrs + [__file__], obj):
            jobs.append((f, [CXX, "-O3", "-std=c++17", "-fPIC", "-ffp-contract=off",
                             "-fno-fast-math", "-pthread", "-c", src, "-o", obj]))
    # translation units compile in parallel (the slowest, primal.cu, first)
    from concurrent.futures import ThreadPoolExecutor

    jobs.sort(key=lambda j: j[0] != "primal.cu")
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for f, _ in zip([j[0] for j in jobs],
                        list(ex.map(lambda j: _run(j[1], os.path.join(OBJ, j[0] + ".log")),
                                    jobs))):
            if verbose:
                print("built", f)
    if force or _newer(objs, LIB):
        _run([NVCC, "-shared"] + ARCH + ["-o", LIB] + objs + ["-lpthread"],
             os.path.join(OBJ, "link.log"))
        if verbose:
            print("linked", LIB)
    build_torch_ext(force, verbose)
    return LIB


TORCH_EXT = os.path.join(HERE, "libgridot_torch.so")


def build_torch_ext(force: bool = False, verbose: bool = False) -> str | None:
    """The PyTorch extension (torch_ops.cpp) that loads libgridot_b200.so as a
    linked dependency and registers torch.ops.gridot_b200.*; g++ against the
    installed torch headers, rpath $ORIGIN so the two libraries travel together."""
    src = os.path.join(HERE, "torch_ops.cpp")
    hdr = os.path.join(REPO, "include", "gridot_b200.h")
    if not (force or _newer([src, hdr, LIB, __file__], TORCH_EXT)):
        return TORCH_EXT
    try:
        import torch
        from torch.utils import cpp_extension
    except Exception:  # pragma: no cover - torch is part of the image
        return None
    inc = []
    for pth in cpp_extension.include_paths():
        inc += ["-I", pth]
    cuda_home = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    libdir = os.path.join(os.path.dirname(torch.__file__), "lib")
    abi = int(torch._C._GLIBCXX_USE_CXX11_ABI)
    _run([CXX, "-O2", "-std=c++17", "-fPIC", "-shared", src] + inc +
         ["-I", os.path.join(cuda_home, "include"), f"-D_GLIBCXX_USE_CXX11_ABI={abi}",
          "-L", libdir, "-ltorch", "-ltorch_cpu", "-lc10", "-lc10_cuda", "-ltorch_cuda",
          "-L", HERE, "-lgridot_b200", "-Wl,-rpath,$ORIGIN", "-o", TORCH_EXT],
         os.path.join(OBJ, "torch_ops.log"))
    if verbose:
        print("built", TORCH_EXT)
    return TORCH_EXT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
