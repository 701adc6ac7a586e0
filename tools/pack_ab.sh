#!/bin/bash
# Activation-pack variants: per-kernel launch list of one bench step each.
mkdir -p gpurun_out/pack
for v in 32 64 128; do
  DNNP_PACK_PIX=$v ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/pack/l$v.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
done
