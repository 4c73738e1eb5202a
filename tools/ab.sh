#!/bin/bash
# build libsdas.so from git revision $1 (default HEAD) as paper_2601_03197_b200/libsdas_A.so, for
# same-box A/B timing:  SDAS_LIB=$PWD/paper_2601_03197_b200/libsdas_A.so python bench.py ...
REV=${1:-HEAD}
rm -rf /tmp/ab_src && mkdir -p /tmp/ab_src
git -C /root/repo archive "$REV" paper_2601_03197_b200 include | tar -x -C /tmp/ab_src
SDAS_LIB=/root/repo/paper_2601_03197_b200/libsdas_A.so python /tmp/ab_src/paper_2601_03197_b200/build.py --force
