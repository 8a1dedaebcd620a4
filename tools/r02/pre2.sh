set -u
O=gpurun_out/r02c; mkdir -p $O
PERMB200_TOL_REPORT=$O/tol_report.json timeout 1200 python -m pytest tests/test_gpu_orders.py tests/test_bench_launch.py tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_concurrency.py tests/test_gpu_runner.py tests/test_abi.py -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?" > $O/status.txt
timeout 300 python tools/r02/m1_plans.py > $O/m1_plans_glynn.log 2>&1; echo "m1g rc=$?" >> $O/status.txt
timeout 300 python tools/r02/m1_plans.py --alg ryser > $O/m1_plans_ryser.log 2>&1; echo "m1r rc=$?" >> $O/status.txt
timeout 600 python tools/r02/batched_run.py --out $O/batched.json > $O/batched.log 2>&1; echo "batched rc=$?" >> $O/status.txt
timeout 600 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench rc=$?" >> $O/status.txt
PERMB200_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 2 --warmup 3 > $O/bench_gloo2.json 2> $O/bench_gloo2.err; echo "bench2 rc=$?" >> $O/status.txt
timeout 900 python tools/r02/table_av.py --out $O/r02_precision > $O/table_av.log 2>&1; echo "tableav rc=$?" >> $O/status.txt
for v in 00 10 01 11 00 10 01 11; do echo "variant $v" >> $O/sweep_variants.log; timeout 120 tools/microbench/sweep_bench_$v 8 >> $O/sweep_variants.log 2>&1; done
