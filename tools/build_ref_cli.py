"""Builds the REFERENCE's evaluation CLI (/root/reference/proj/tools/xigemm_bench.cpp,
unchanged) twice, with the CLI11 shim (tools/cli11_shim):

  build/ref_cli/xigemm-bench      against this library (include/xigemm + libxigemm_b200.so)
  build/ref_cli/xigemm-bench-ref  against the reference itself (oracle/_ref, namespace
                                  renamed xigemm_ref as in oracle/Makefile)

Same source, same flags: running both with identical arguments shows the
drop-in at the level of a real caller (tests/test_reference_cli.py compares
their CSV output).  Nothing is copied into the repository."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "/root/reference/proj/tools/xigemm_bench.cpp"
REF_INC = "/root/reference/proj/include"
OUT = os.path.join(ROOT, "build", "ref_cli")
LIB_DIR = os.path.join(ROOT, "paper_2403_06924_b200", "lib")
REF_DIR = os.path.join(ROOT, "oracle", "_ref")


def main() -> int:
    if not os.path.exists(SRC):
        print("reference CLI absent; nothing to build")
        return 0
    os.makedirs(OUT, exist_ok=True)
    shim = os.path.join(ROOT, "tools", "cli11_shim")
    common = ["g++", "-O2", "-std=gnu++20", "-I", shim]
    ours = common + ["-I", os.path.join(ROOT, "include"), SRC, "-o", os.path.join(OUT, "xigemm-bench"),
                     "-L", LIB_DIR, "-lxigemm_b200", f"-Wl,-rpath,{LIB_DIR}",
                     "-Wl,-rpath,$ORIGIN/../../paper_2403_06924_b200/lib"]
    ref = common + ["-Dxigemm=xigemm_ref", "-I", REF_INC, SRC, "-o", os.path.join(OUT, "xigemm-bench-ref"),
                    "-L", REF_DIR, "-lxigemm_ref", f"-Wl,-rpath,{REF_DIR}",
                    "-Wl,-rpath,$ORIGIN/../../oracle/_ref"]
    rc = 0
    for cmd in (ours, ref):
        if cmd is ref and not os.path.exists(os.path.join(REF_DIR, "libxigemm_ref.so")):
            continue
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            print("FAILED:", " ".join(cmd), "\n", r.stderr[-4000:])
            rc = 1
        else:
            print("built", cmd[cmd.index("-o") + 1])
    return rc


if __name__ == "__main__":
    sys.exit(main())
