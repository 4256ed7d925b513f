#!/bin/bash
for v in main n2v5 claim16 claim64; do
  if [ $v = main ]; then export WF_LIB=paper_2107_11983_b200/libwalkforge_b200.so; else export WF_LIB=tools/_exp_$v/libwf.so; fi
  echo "== $v c2"; python tools/profile_walk.py --config c2 --launches 4 --flush 2>&1 | tail -1
  echo "== $v c2 counts"; python tools/profile_walk.py --config c2 --launches 4 --flush --counts 2>&1 | tail -1
  echo "== $v c2 4M"; python tools/profile_walk.py --config c2 --launches 4 --flush --queries 4194304 2>&1 | tail -1
  echo "== $v c1"; python tools/profile_walk.py --config c1 --launches 4 --flush 2>&1 | tail -1
  echo "== $v c4"; python tools/profile_walk.py --config c4 --launches 3 2>&1 | tail -1
  echo "== $v c3"; python tools/profile_walk.py --config c3 --launches 3 2>&1 | tail -1
done
