#!/bin/bash
# rebuild libsdas.so with -Xptxas -v and print registers / spills per K1 instantiation (TRACE, MAXOUT, CLS)
cd "$(dirname "$0")/.." || exit 1
python paper_2601_03197_b200/build.py --force -v 2>&1 | awk '
  /Compiling entry function/ && /k1_simulate/ { match($0, /k1_simulateILb[01]ELi[12]ELb[01]ELi[012]/); name = substr($0, RSTART + 11, RLENGTH - 11); next }
  name && /spill stores/ { sp = $0; sub(/^ */, "", sp) }
  name && /Used [0-9]+ registers/ { match($0, /Used [0-9]+ registers/); print name, substr($0, RSTART, RLENGTH), "|", sp; name = "" }'
