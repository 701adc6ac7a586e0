#!/bin/bash
# Under gpurun: find the bench's dominant kernel, then capture it once with
# ncu --set full (one GPU, single process) and also take the bench launch list.
#   bash tools/capture_dominant.sh <tag>
set -u
TAG=${1:-dom}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 600 python bench.py --no-cpu --no-e2e --no-sustained --no-bw --no-sweep --steps 5 > "$OUT/bench.json" 2> "$OUT/bench.err"
read -r LAYER PASS KRE < <(python3 - "$OUT/bench.json" <<'EOF'
import json, sys
d = json.load(open(sys.argv[1]))
name = d["roofline"]["kernel"]
layer, pas = name.split(".")
kre = "wgrad_tma" if pas == "bwd_filter" else "conv_tma"
print(layer, pas, kre)
EOF
)
echo "dominant: $LAYER $PASS ($KRE)" > "$OUT/dominant.txt"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$KRE" -s 2 -c 1 \
  -o "$OUT/prof_${LAYER}_${PASS}" python tools/prof_layer.py "$LAYER" "$PASS" 3 > "$OUT/ncu_full.log" 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-sustained --no-bw --no-sweep \
  > "$OUT/ncu_bench.log" 2>&1
# keep the artefacts small enough to copy back: CSV pages of the capture
for REP in "$OUT"/prof_*.ncu-rep; do
  ncu -i "$REP" --page details --csv > "${REP%.ncu-rep}_details.csv" 2>/dev/null
  ncu -i "$REP" --page raw --csv > "${REP%.ncu-rep}_raw.csv" 2>/dev/null
  [ -n "${KEEP_REP:-}" ] || rm -f "$REP"
done
cat "$OUT/dominant.txt"
