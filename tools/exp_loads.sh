#!/bin/bash
# A/B of the random-gather load flavour (tools/_exp_*/libwf.so built with -DWF_LDR=...)
for n in cg nc na pl; do
  for L in 0 1; do
    echo "== $n layout=$L c5/s24"; WF_LIB=tools/_exp_$n/libwf.so python tools/profile_walk.py --config c5 --scale 24 --launches 3 --layout $L 2>&1 | tail -1
  done
  echo "== $n c3"; WF_LIB=tools/_exp_$n/libwf.so python tools/profile_walk.py --config c3 --launches 3 2>&1 | tail -1
  echo "== $n c4"; WF_LIB=tools/_exp_$n/libwf.so python tools/profile_walk.py --config c4 --launches 3 2>&1 | tail -1
done
