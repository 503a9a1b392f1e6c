mkdir -p gpurun_out/q7
timeout 900 python -m pytest tests -m gpu -q -x -k "set_grads or sharding or graph_equals or trajectory or dshard or clustered or host" > gpurun_out/q7/pytest.log 2>&1; echo "exit $?" >> gpurun_out/q7/pytest.log
for C in C4 S1; do timeout 300 python bench.py --config $C --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/q7/bench_$C.json 2>&1; done
