#!/usr/bin/env python
"""Run bench.py's serving-replay line alone (diagnostic, one GPU)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench

    sys.argv = [sys.argv[0]]
    args = bench.parse()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    print(json.dumps(bench.serving_replay(args, dev)))


if __name__ == "__main__":
    main()
