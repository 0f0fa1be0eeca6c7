#!/bin/bash
# Run on the GPU box (gpurun): quick parity subset, then one ncu --set full
# capture of the kernels matching $1 on config $2 (default C3).
#   gpurun -- 'bash tools/prof_kernels.sh "k_c_|k_t_" C3 name'
set -u
K=${1:-k_c_}; CFG=${2:-C3}; NAME=${3:-prof}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "c2_full or c3 or c4 or edge or geometries" > gpurun_out/gputest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/gputest.log
python tools/scale_prof.py $CFG > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"$K" -c ${4:-6} -o gpurun_out/$NAME \
  python tools/scale_prof.py $CFG > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?"
