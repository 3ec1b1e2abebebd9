"""Build an A/B variant of the library with extra nvcc defines (kernel experiments).

  python tools/build_variant.py TAG -DMCP_K1S_PAIRS=7 ...
writes paper_1911_03813_b200/_lib/variants/libmomentcp_b200_TAG.so; select it at run time with
MCP_LIBRARY=<path>.  The product build is __graft_entry__.build().
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as ge  # noqa: E402


def main():
    tag, defs = sys.argv[1], sys.argv[2:]
    out_dir = os.path.join(ge.PKG, "_lib", "variants", tag)
    os.makedirs(out_dir, exist_ok=True)
    objs, procs = [], []
    for src in ge.SOURCES:
        obj = os.path.join(out_dir, src.replace(".cu", ".o"))
        flags = [f for f in ge.NVCC_FLAGS if f != "-shared"]
        procs.append(subprocess.Popen([ge._nvcc(), *flags, *defs, "-c", os.path.join(ge.CSRC, src),
                                       "-o", obj], stdout=subprocess.DEVNULL,
                                      stderr=subprocess.DEVNULL))
        objs.append(obj)
    if any(p.wait() for p in procs):
        raise SystemExit("nvcc failed")
    lib = os.path.join(ge.PKG, "_lib", "variants", f"libmomentcp_b200_{tag}.so")
    subprocess.check_call([ge._nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                           "-Xcompiler", "-fPIC", *objs, "-o", lib])
    print(lib)


if __name__ == "__main__":
    main()
