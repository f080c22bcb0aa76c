#!/bin/bash
# Build an A/B variant of libcatgnn.so with extra nvcc defines into
# paper_2404_02300_b200/build/variants/<name>/libcatgnn.so (load with CATGNN_LIB=...).
#   scripts/build_variant.sh NAME "-DAGG_NARROW_UNROLL=8 -DAGG_NARROW_MINB=3"
set -e
name=$1; defs=$2
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/paper_2404_02300_b200/build/variants/$name
rm -rf "$out"; mkdir -p "$out"
cp -r "$root/paper_2404_02300_b200/csrc" "$out/csrc"
python3 - "$root" "$out" "$defs" <<'PY'
import sys
root, out, defs = sys.argv[1:4]
s = open(f"{root}/paper_2404_02300_b200/Makefile").read()
s = s.replace("$(CURDIR)/../include", f"{root}/include").replace("../include/catgnn.h", f"{root}/include/catgnn.h")
s = s.replace("NVFLAGS  := ", f"NVFLAGS  := {defs} ", 1)
open(f"{out}/Makefile", "w").write(s)
PY
make -C "$out" -j8 libcatgnn.so > "$out/build.log" 2>&1 || { tail -20 "$out/build.log"; exit 1; }
echo "$out/libcatgnn.so"
