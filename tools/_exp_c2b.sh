#!/bin/bash
echo "== c2 flush"; python tools/profile_walk.py --config c2 --launches 4 --flush 2>&1 | tail -1
echo "== c2 flush counts"; python tools/profile_walk.py --config c2 --launches 4 --flush --counts 2>&1 | tail -1
echo "== c2 diag"; WF_LIB=tools/_exp_diag/libwf.so python tools/profile_walk.py --config c2 --launches 4 --flush --diag-times 2>&1 | tail -2
echo "== c2 diag 4M"; WF_LIB=tools/_exp_diag/libwf.so python tools/profile_walk.py --config c2 --launches 4 --flush --diag-times --queries 4194304 2>&1 | tail -2
echo "== c1 diag"; WF_LIB=tools/_exp_diag/libwf.so python tools/profile_walk.py --config c1 --launches 4 --flush --diag-times 2>&1 | tail -2
echo "== c4 diag"; WF_LIB=tools/_exp_diag/libwf.so python tools/profile_walk.py --config c4 --launches 3 --diag-times 2>&1 | tail -2
echo "== c3 diag"; WF_LIB=tools/_exp_diag/libwf.so python tools/profile_walk.py --config c3 --launches 3 --diag-times 2>&1 | tail -2
