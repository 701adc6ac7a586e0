#!/bin/bash
# DRAM bytes and duration of every kernel of one bench step (ncu, serialised,
# cold caches): per-op traffic vs the op's algorithmic bytes.
#   bash tools/op_traffic.sh <tag>
OUT=gpurun_out/${1:-traffic}
mkdir -p "$OUT"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file "$OUT/launches_dram.csv" \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-sustained --no-bw --no-sweep \
  > "$OUT/ncu_bench.log" 2>&1
echo "ncu rc=$?"
