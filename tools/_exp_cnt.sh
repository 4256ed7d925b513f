#!/bin/bash
echo "== main c2"; python tools/profile_walk.py --config c2 --launches 4 --flush 2>&1 | tail -1
echo "== main c2 counts"; python tools/profile_walk.py --config c2 --launches 4 --flush --counts 2>&1 | tail -1
echo "== main c1"; python tools/profile_walk.py --config c1 --launches 4 --flush 2>&1 | tail -1
echo "== main c4"; python tools/profile_walk.py --config c4 --launches 3 2>&1 | tail -1
echo "== main c3"; python tools/profile_walk.py --config c3 --launches 3 2>&1 | tail -1
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py > gpurun_out/run32_bench.json 2>gpurun_out/run32_bench.err; cat gpurun_out/run32_bench.json
