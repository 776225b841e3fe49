#!/bin/bash
# A/B of two builds of the library on one box, alternating processes:
#   bash scripts/ab_lib.sh alt/libhmat_prev.so "c4:WARM=30,REPS=10,NRHS=8" "c2:WARM=100,REPS=40,NRHS=4" ...
# (B = the in-tree libhmat.so; A = the given build, loaded through HMAT_LIB_AB)
set -u
ALT=$1
shift
for rep in 1 2 3; do
  for spec in "$@"; do
    cfg=${spec%%:*}
    set_=${spec#*:}
    echo -n "new  "; python scripts/kernel_sweep.py $cfg "$set_" 2>&1 | grep -v Warn | tail -1
    echo -n "prev "; HMAT_LIB_AB=$ALT python scripts/kernel_sweep.py $cfg "$set_" 2>&1 | grep -v Warn | tail -1
  done
done
