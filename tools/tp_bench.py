#!/usr/bin/env python
"""Run bench.py's config-4 (70B, TP=8) line alone on one GPU (diagnostic)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench

    args = bench.parse.__wrapped__() if hasattr(bench.parse, "__wrapped__") else None
    sys.argv = [sys.argv[0]]
    args = bench.parse()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    print(json.dumps(bench.tp_config(args, dev, 1, 0)))


if __name__ == "__main__":
    main()
