#!/bin/bash
# round 2, first box call: slot kernel parity + A/B against the round-1 default, full GPU suite
o=gpurun_out/r02a; mkdir -p $o
nvidia-smi > $o/smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "slot or invariance_auto" > $o/pytest_slot.txt 2>&1
timeout 900 python bench.py --no-cpu --steps 5 --warmup 3 > $o/bench_slots.json 2> $o/bench_slots.err
timeout 900 python bench.py --no-cpu --steps 5 --warmup 3 --layout blocked > $o/bench_blocked.json 2> $o/bench_blocked.err
timeout 1500 python -m pytest tests/ -x -q -m gpu > $o/pytest_gpu.txt 2>&1
