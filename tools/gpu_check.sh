#!/bin/bash
# One gpurun call: GPU tests, the bench line, the launch list and one full ncu
# capture of a chosen kernel.  Usage (under gpurun):
#   bash tools/gpu_check.sh <tag> [layer pass kernel-regex]
set -u
TAG=${1:-run}
LAYER=${2:-conv1}
PASS=${3:-fwd}
KRE=${4:-conv_tc}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > "$OUT/gpu.txt" 2>&1
nproc >> "$OUT/gpu.txt"; lscpu | grep -E "Model name|^CPU\(s\)" >> "$OUT/gpu.txt"
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest exit $?" >> "$OUT/pytest_gpu.log"
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
  echo "smoke exit $?" >> "$OUT/smoke.log"
fi
timeout 600 python bench.py ${BENCH_ARGS:-} > "$OUT/bench.json" 2> "$OUT/bench.err"
echo "bench exit $?" >> "$OUT/bench.err"
if [ "${SKIP_NCU:-0}" != 1 ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu \
    > "$OUT/ncu_bench.log" 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$KRE" -s 2 -c 1 \
    -o "$OUT/prof_${LAYER}_${PASS}" python tools/prof_layer.py "$LAYER" "$PASS" 3 \
    > "$OUT/ncu_full.log" 2>&1
fi
tail -3 "$OUT/pytest_gpu.log" 2>/dev/null
cat "$OUT/bench.json"
