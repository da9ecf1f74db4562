#!/bin/bash
# Quick C5 check on the GPU box: parity of the 3-D second-order path (scaled and
# full size) and operator timings.  usage: tools/quick_c5.sh TAG [ops]
TAG=${1:-x}; OPS=${2:-gradient,residual2,jacobian,matvec}
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "C5" > gpurun_out/q_${TAG}_test.log 2>&1
echo rc=$? >> gpurun_out/q_${TAG}_test.log
python tools/time_ops.py 4 --ops $OPS --reps 5 > gpurun_out/q_${TAG}_time.log 2>&1
