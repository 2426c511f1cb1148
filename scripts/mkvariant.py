"""Build an experiment variant of the library: a git revision's sources plus selected pieces of the
working tree, into paper_2005_07547_b200/lib/variants/<name>/ (picked at run time with
PSTF_LIB_PATH; see scripts/gpu_ab.sh).  Used to bisect performance changes on the GPU box.

  python scripts/mkvariant.py NAME CHANGES [REV]      CHANGES: comma list of
      keys     working-tree pstf_keys.cuh           fin      working-tree finite3()
      nosleep  drop the mbarrier back-off sleep     dedup    working-tree tile loop (one body)
      all      the whole working tree               none     REV as is
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = "paper_2005_07547_b200/csrc"


def seg(text, a, b):
    i = text.index(a)
    j = text.index(b, i)
    return text[i:j + len(b)]


def main():
    name, changes = sys.argv[1], sys.argv[2].split(",")
    rev = sys.argv[3] if len(sys.argv) > 3 else "HEAD"
    d = f"/tmp/pstf_var_{name}"
    shutil.rmtree(d, ignore_errors=True)
    os.makedirs(d)
    arch = subprocess.run(["git", "-C", ROOT, "archive", rev, CSRC, "include"], capture_output=True,
                          check=True).stdout
    subprocess.run(["tar", "-x", "-C", d], input=arch, check=True)
    if "all" in changes:
        shutil.rmtree(f"{d}/{CSRC}")
        shutil.copytree(f"{ROOT}/{CSRC}", f"{d}/{CSRC}")
        shutil.copy(f"{ROOT}/include/pstf_field.h", f"{d}/include/pstf_field.h")
    cur = open(f"{ROOT}/{CSRC}/field.cu").read()
    f = f"{d}/{CSRC}/field.cu"
    s = open(f).read()
    if "keys" in changes:
        shutil.copy(f"{ROOT}/{CSRC}/pstf_keys.cuh", f"{d}/{CSRC}/pstf_keys.cuh")
    if "fin" in changes:
        a = "__device__ __forceinline__ bool finite3"
        s = s.replace(seg(s, a, "}\n"), seg(cur, a, "}\n"))
    if "nosleep" in changes:
        s = s.replace("        __nanosleep(64); /* back off: leave issue slots to the other CTAs on the SM */\n", "")
    if "dedup" in changes:
        old = seg(s, "    uint32_t it = 0;\n    for (uint64_t tile", "        vertex_body(a, src, live, sm);\n    }\n}")
        new = seg(cur, "    uint32_t it = 0;\n    const uint64_t ntiles", "\n    }\n}")
        new = new.replace("policy, lane)", "policy)").replace("gridDim.x, lane)", "gridDim.x)")
        new = new.replace("tid < 32 && nt", "tid == 0 && nt")
        s = s.replace(old, new)
    open(f, "w").write(s)
    out = f"{ROOT}/paper_2005_07547_b200/lib/variants/{name}"
    os.makedirs(out, exist_ok=True)
    cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
           "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
           "--expt-relaxed-constexpr", "-cudart", "static", "-Xptxas", "-v", "-shared", "-o",
           f"{out}/libpstf_b200.so", f] + os.environ.get("VFLAGS", "").split()
    r = subprocess.run(cmd, capture_output=True, text=True)
    open(f"{out}/ptxas.log", "w").write(r.stderr)
    if r.returncode:
        print(r.stderr[-3000:])
        sys.exit(1)
    size = subprocess.run([sys.executable, f"{ROOT}/scripts/sass_size.py", f"{out}/libpstf_b200.so",
                           "tiledILi1"], capture_output=True, text=True).stdout.strip()
    print(name, size)


if __name__ == "__main__":
    main()
