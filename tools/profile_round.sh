#!/bin/bash
# Run on the GPU box (gpurun): bench line, launch list, full captures of the
# dominant compress / decompress kernels at the metric's configuration (C5).
# Outputs under gpurun_out/; summarise here with tools/launches.py and
# tools/ncu_summary.py, then copy into profiles/ (see profiles/README.md).
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
echo "bench rc=$?"
tail -1 gpurun_out/bench.log > gpurun_out/bench.json
# every launch of one compress + one decompress step (cold, serialised: shares, not absolutes)
timeout 900 python bench.py --warmup 0 --profile-steps 1 --no-cpu-baseline --no-e2e > gpurun_out/plain_prof.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --warmup 0 --profile-steps 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
# the dominant kernels, one launch each (C5 through tools/scale_prof.py)
python tools/scale_prof.py C5 > gpurun_out/plain5.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:"k_c_mainILi3ELi0ELb1|k_c_write|k_stats|k_d_decode|k_d_reconILi3" -c 5 -o gpurun_out/full_c5 \
  python tools/scale_prof.py C5 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
# the e2e path against the box's PCIe ceiling, and the other BASELINE configs
{ python tools/pcie_duplex.py 4.41 8.59; python tools/e2e_check.py --check --steps 2; } > gpurun_out/e2e.txt 2>&1
{ for c in C1 C2 C3 C4; do python tools/scale_check.py $c | tail -3; done; python tools/path_cross.py; GEN=C4 python tools/path_cross.py 50000x500; } > gpurun_out/configs.txt 2>&1
ls -la gpurun_out
