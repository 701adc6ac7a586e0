#!/bin/bash
# Under gpurun: refresh every measurement the docs cite (tests, bench, CLI
# suites, bandwidth ops, accuracy, ncu of the dominant kernel + launch list).
#   bash tools/round_refresh.sh <tag>
set -u
TAG=${1:-refresh}
OUT=gpurun_out/$TAG
mkdir -p "$OUT/cli"
timeout 900 python -m pytest tests -q -m gpu > "$OUT/pytest_gpu.txt" 2>&1
tail -3 "$OUT/pytest_gpu.txt"
timeout 600 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 600 python bench.py --impl reference > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
for s in table2 alexnet overfeat_vgg; do
  timeout 600 python -m paper_1410_0759_b200.bench_cli run --suite $s --passes fwd,bwd_data,bwd_filter \
    --repeats 5 --peak 856250 --format csv,json --out "$OUT/cli/$s.csv" --quiet > "$OUT/cli/$s.txt" 2>&1
  echo "rc=$?" >> "$OUT/cli/$s.txt"
done
timeout 600 python -m paper_1410_0759_b200.bench_cli run --suite table2 --passes fwd,bwd_data,bwd_filter \
  --verify --quiet --out "$OUT/cli/table2_verify.csv" > "$OUT/cli/table2_verify.txt" 2>&1
echo "rc=$?" >> "$OUT/cli/table2_verify.txt"
timeout 600 python -m paper_1410_0759_b200.bench_cli run --suite table2 --dtype f64 --batch 16 \
  --passes fwd,bwd_data,bwd_filter --quiet --out "$OUT/cli/table2_f64.csv" > "$OUT/cli/table2_f64.txt" 2>&1
timeout 600 python -m paper_1410_0759_b200.bench_cli sweep --suite overfeat_vgg --layer of_conv3 \
  --batches 1,2,4,8,16,32,64,128,256 --passes fwd,bwd_data,bwd_filter --quiet \
  --out "$OUT/cli/sweep_of_conv3.csv" > "$OUT/cli/sweep_of_conv3.txt" 2>&1
timeout 600 python tools/bench_bw.py --json "$OUT/bandwidth_ops.json" > "$OUT/bandwidth_ops.txt" 2>&1
timeout 600 python tools/accuracy_probe.py > "$OUT/accuracy_probe.txt" 2>&1
timeout 300 python tools/explicit_control.py > "$OUT/explicit_negative_control.txt" 2>&1
timeout 300 python tools/fused_probe.py > "$OUT/fused_epilogue_probe.txt" 2>&1
bash tools/capture_dominant.sh "$TAG/dom" > "$OUT/capture.txt" 2>&1
echo done
