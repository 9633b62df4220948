#!/bin/bash
# Build the library of git revision REV into alt_lib/REV/ (A/B runs: KRUL_LIB=alt_lib/REV/libkrul_b200.so)
REV=$1
D=$(mktemp -d)
git archive $REV paper_2507_08045_b200/csrc include | tar -x -C $D
make -s -j16 -C $D/paper_2507_08045_b200/csrc >/dev/null
mkdir -p alt_lib/$REV
cp $D/paper_2507_08045_b200/_lib/libkrul_b200.so alt_lib/$REV/
rm -rf $D
echo alt_lib/$REV/libkrul_b200.so
