"""Compiles the REFERENCE's own doctest suites (/root/reference/proj/tests)
against this library's drop-in headers (include/xigemm) and
paper_2403_06924_b200/lib/libxigemm_b200.so — the drop-in proof.

Nothing is copied into the repository: sources are read from the reference
tree at build time; binaries go to build/ref_suites/ (git-ignored, they travel
to the GPU box with the snapshot).  test_pipeline.cpp does not compile on GCC 13
as written (unqualified xigemm(...) is ambiguous with the namespace, see
SURVEY.md §4); the same mechanical qualification the survey used is applied to
a build-time temporary.
"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = "/root/reference/proj/tests"
OUT = os.path.join(ROOT, "build", "ref_suites")
LIB_DIR = os.path.join(ROOT, "paper_2403_06924_b200", "lib")


def main() -> int:
    if not os.path.isdir(REF_TESTS):
        print("reference tests absent; nothing to build")
        return 0
    os.makedirs(OUT, exist_ok=True)
    rc = 0
    for f in sorted(os.listdir(REF_TESTS)):
        if not (f.startswith("test_") and f.endswith(".cpp")):
            continue
        src = os.path.join(REF_TESTS, f)
        text = open(src).read()
        if f == "test_pipeline.cpp":
            text = re.sub(r"([^:A-Za-z_])xigemm\(", r"\1xigemm::xigemm(", text)
        tmp = os.path.join(OUT, f)
        with open(tmp, "w") as fh:
            fh.write(text)
        exe = os.path.join(OUT, f[:-4])
        cmd = ["g++", "-O1", "-std=gnu++20", "-I", os.path.join(ROOT, "tools", "doctest_shim"),
               "-I", os.path.join(ROOT, "include"), "-I", REF_TESTS, tmp, "-o", exe,
               "-L", LIB_DIR, "-lxigemm_b200", f"-Wl,-rpath,{LIB_DIR}", "-Wl,-rpath,$ORIGIN/../../paper_2403_06924_b200/lib"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            print(f"FAILED {f}:\n{r.stderr[-3000:]}")
            rc = 1
        else:
            print(f"built {exe}")
        os.remove(tmp)
    return rc


if __name__ == "__main__":
    sys.exit(main())
