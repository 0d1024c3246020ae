"""Write tests/golden/metrics_records.json: the reference's run_records for a
fixed 3-mode / 3-device run (imports the reference from /root/reference; run
in the build container only -- the fixture is committed)."""

import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
import shardkrp.metrics as R  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sample(mod):
    ms = [mod.ModeMetrics(d, [0.1 * d + 0.01, 0.2, 0.05 * (d + 1)], [10 + d, 20, 30], [1, 2, 3],
                          staging_bytes=5 * d, staging_seconds=0.1, allgather_bytes=7, allgather_seconds=0.2 * d,
                          barrier_count=d, wall_seconds=0.3) for d in range(3)]
    return mod.RunMetrics(3, ms, [0.5, 0.25, 0.125], 1.5)


class Platform:
    devices, workers_per_device, column_width, rank, accumulation, scheduling = 3, 1, 32, 16, "atomic", "dynamic"


class Tensor:
    name, shape, nnz = "golden", (3, 4, 5), 60


if __name__ == "__main__":
    with open(os.path.join(HERE, "metrics_records.json"), "w") as fh:
        json.dump(R.run_records(sample(R), Platform, Tensor), fh, indent=1)
