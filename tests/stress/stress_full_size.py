"""Full-size determinism: configs 4 and 5 at their BASELINE object counts, every output of
repeated predicts compared with the first run's (the bench line verifies ~65k sampled rows)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from stress_determinism import run  # noqa: E402

from paper_2211_00391_b200 import synthetic  # noqa: E402

if __name__ == "__main__":
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    run("K2w config 4, 8M objects", synthetic.CONFIGS[4], iters)
    run("K5 config 5, 16M objects", synthetic.CONFIGS[5], max(2, iters // 2))
    W = synthetic.WorkloadSpec
    run("K5 fp16 config 5, 16M objects", W(**{**synthetic.CONFIGS[5].__dict__, "half_leaves": True}), max(2, iters // 2), half=True)
