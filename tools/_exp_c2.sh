#!/bin/bash
for q in 65536 1048576 4194304; do
  for L in 0 8; do
    echo "== q=$q layout=$L flush"; python tools/profile_walk.py --config c2 --queries $q --layout $L --launches 4 --flush 2>&1 | tail -2
  done
done
echo "== nc c2"; WF_LIB=tools/_exp_nc/libwf.so python tools/profile_walk.py --config c2 --launches 4 --flush 2>&1 | tail -1
echo "== nc c4"; WF_LIB=tools/_exp_nc/libwf.so python tools/profile_walk.py --config c4 --launches 3 2>&1 | tail -1
echo "== cg c4"; python tools/profile_walk.py --config c4 --launches 3 2>&1 | tail -1
echo "== nc c5s24"; WF_LIB=tools/_exp_nc/libwf.so python tools/profile_walk.py --config c5 --scale 24 --launches 3 2>&1 | tail -1
echo "== cg c5s24"; python tools/profile_walk.py --config c5 --scale 24 --launches 3 2>&1 | tail -1
