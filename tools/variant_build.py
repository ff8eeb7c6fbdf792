"""Build an A/B variant of libisogs.so: one translation unit recompiled with
extra nvcc flags, linked with the current objects of the others.

    python tools/variant_build.py NAME FILE.cu -DFOO=1 ...
    -> paper_2509_05216_b200/_build/NAME/libisogs.so  (ISOGS_LIB=... to use it)
"""

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2509_05216_b200 import build as B  # noqa: E402


def main():
    name, src, flags = sys.argv[1], sys.argv[2], sys.argv[3:]
    B.build()
    out = os.path.join(B.OUT_DIR, name)
    os.makedirs(out, exist_ok=True)
    obj = os.path.join(out, src.replace(".cu", ".o"))
    # VARIANT_SRC=path compiles another copy of the file (e.g. `git show HEAD:...`)
    path = os.environ.get("VARIANT_SRC") or os.path.join(B.CSRC, src)
    cmd = [B.nvcc(), *B.ARCH, *B.COMMON, "-I" + B.CSRC, *B.SOURCES[src], *flags, "-c", path,
           "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stderr)
    with open(obj + ".ptxas.txt", "w") as fh:
        fh.write(r.stderr)
    objs = [obj] + [os.path.join(B.OUT_DIR, s.replace(".cu", ".o")) for s in B.SOURCES if s != src]
    lib = os.path.join(out, "libisogs.so")
    r = subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", lib, *objs, "-cudart", "static"],
                       capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stderr)
    print(lib)


if __name__ == "__main__":
    main()
