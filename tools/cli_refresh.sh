#!/bin/bash
# Under gpurun: the bench CLI over the bundled suites (all passes), verify,
# f64 and the OverFeat sweep, plus the accuracy probe.
#   bash tools/cli_refresh.sh <tag>
OUT=gpurun_out/${1:-cli}
mkdir -p "$OUT"
for s in table2 alexnet overfeat_vgg; do
  timeout 600 python -m paper_1410_0759_b200.bench_cli run --suite $s --passes fwd,bwd_data,bwd_filter \
    --repeats 5 --peak 856250 --format csv,json --out "$OUT/$s.csv" --quiet > "$OUT/$s.txt" 2>&1
  echo "rc=$?" >> "$OUT/$s.txt"
done
timeout 600 python -m paper_1410_0759_b200.bench_cli run --suite table2 --passes fwd,bwd_data,bwd_filter \
  --verify --quiet --out "$OUT/table2_verify.csv" > "$OUT/table2_verify.txt" 2>&1
echo "rc=$?" >> "$OUT/table2_verify.txt"
timeout 600 python -m paper_1410_0759_b200.bench_cli run --suite table2 --dtype f64 --batch 16 \
  --passes fwd,bwd_data,bwd_filter --quiet --out "$OUT/table2_f64.csv" > "$OUT/table2_f64.txt" 2>&1
timeout 600 python -m paper_1410_0759_b200.bench_cli sweep --suite overfeat_vgg --layer of_conv3 \
  --batches 1,2,4,8,16,32,64,128,256 --passes fwd,bwd_data,bwd_filter --quiet \
  --out "$OUT/sweep_of_conv3.csv" > "$OUT/sweep_of_conv3.txt" 2>&1
timeout 600 python tools/accuracy_probe.py > "$OUT/accuracy_probe.txt" 2>&1
