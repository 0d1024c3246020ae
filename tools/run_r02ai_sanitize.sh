#!/bin/bash
# compute-sanitizer memcheck + racecheck on the round-2 kernels (fiber metadata ring, paired groups, cells)
o=gpurun_out/r02ai; mkdir -p $o
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu.py -x -q -k "fiber_odd_tiles and (32-33 or 64-37)" > $o/memcheck_fibers.txt 2>&1; echo "exit $?" >> $o/memcheck_fibers.txt
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu.py -x -q -k "fiber_odd_tiles and 32-100" > $o/racecheck_fibers.txt 2>&1; echo "exit $?" >> $o/racecheck_fibers.txt
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_cells.py -x -q -k "golden and u3" > $o/memcheck_cells.txt 2>&1; echo "exit $?" >> $o/memcheck_cells.txt
