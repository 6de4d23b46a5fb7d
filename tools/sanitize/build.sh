#!/bin/sh
# Builds tools/sanitize/driver against the in-tree library (run from anywhere).
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
ROOT=$(cd "$HERE/../.." && pwd)
LIB="$ROOT/paper_2403_06924_b200/lib"
gcc -O1 -g -std=c11 -I"$ROOT/include" -I/usr/local/cuda/include "$HERE/driver.c" -o "$HERE/driver" \
    -L"$LIB" -lxigemm_b200 -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,'$ORIGIN/../../paper_2403_06924_b200/lib' -Wl,-rpath,/usr/local/cuda/lib64
