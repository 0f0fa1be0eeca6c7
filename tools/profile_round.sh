#!/bin/bash
# Run on the GPU box (gpurun): bench line, launch list, full captures of the
# dominant compress / decompress kernels.  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1
tail -1 gpurun_out/bench.log > gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --warmup 0 --profile-steps 2 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
for k in k_compress_ws k_write_part k_fwd k_quant k_codebook k_decode4 k_reconstruct4 k_inv; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/full_$k \
    python bench.py --warmup 0 --profile-steps 1 --no-cpu-baseline > gpurun_out/ncu_$k.log 2>&1
done
ls -la gpurun_out
