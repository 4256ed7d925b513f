"""Preprocessing (static tables) time of each sampler on a config's graph:

    python tools/pre_time.py [--config c5]

Prints the session's preprocess_seconds (preprocess_static, engine.hpp:190-251)
for ALIAS, ITS and REJ on the weighted DeepWalk program."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    args = ap.parse_args()
    from paper_2107_11983_b200 import abi
    from paper_2107_11983_b200 import engine as E
    from paper_2107_11983_b200.host import DeepWalkProgram, ExecOptions
    cfg = bench.CONFIGS[args.config]
    dg = E.DeviceGraph.rmat(cfg["scale"], 16, seed=1, weighted=True)
    print("graph", dg.info()["V"], dg.info()["E"], "max degree", dg.info()["max_degree"], flush=True)
    for s in (abi.Sampler.ALIAS, abi.Sampler.ITS, abi.Sampler.REJ):
        for rep in range(2):
            sess = E.Session(dg, DeepWalkProgram(80, True), ExecOptions(seed=1, sampler=int(s)))
            print(f"{s.name} preprocess {sess.describe()[2]:.3f} s (run {rep})", flush=True)
            del sess


if __name__ == "__main__":
    main()
