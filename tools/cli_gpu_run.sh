set -x
mkdir -p gpurun_out/cli
python -m pytest tests/test_bench_cli.py -q -m gpu 2>&1 | tail -5
for s in table2 alexnet overfeat_vgg; do
  timeout 600 python -m paper_1410_0759_b200.bench_cli run --suite $s --passes fwd,bwd_data,bwd_filter --repeats 5 --peak 2250000 --format csv,json --out gpurun_out/cli/$s.csv --quiet > gpurun_out/cli/$s.txt 2>&1; echo "rc=$?" >> gpurun_out/cli/$s.txt
done
timeout 300 python -m paper_1410_0759_b200.bench_cli run --suite table2 --passes fwd,bwd_data,bwd_filter --verify --quiet --out gpurun_out/cli/table2_verify.csv > gpurun_out/cli/table2_verify.txt 2>&1; echo "rc=$?" >> gpurun_out/cli/table2_verify.txt
timeout 300 python -m paper_1410_0759_b200.bench_cli run --suite table2 --dtype f64 --batch 16 --passes fwd,bwd_data,bwd_filter --quiet --out gpurun_out/cli/table2_f64.csv > gpurun_out/cli/table2_f64.txt 2>&1; echo "rc=$?" >> gpurun_out/cli/table2_f64.txt
timeout 300 python -m paper_1410_0759_b200.bench_cli sweep --suite overfeat_vgg --layer of_conv3 --batches 1,2,4,8,16,32,64,128,256 --passes fwd,bwd_data,bwd_filter --quiet --out gpurun_out/cli/sweep_of3.csv > gpurun_out/cli/sweep_of3.txt 2>&1; echo "rc=$?" >> gpurun_out/cli/sweep_of3.txt
