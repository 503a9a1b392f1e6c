mkdir -p gpurun_out/g6
timeout 120 ./scripts/micro/tma_store > gpurun_out/g6/tma_store.txt 2>&1
python -c "from paper_2306_06528_b200 import build; build.build()" > gpurun_out/g6/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "set_grads or clustered or bandwidth or sharding or dshard" > gpurun_out/g6/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/g6/pytest.log
python scripts/d_err.py > gpurun_out/g6/derr.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gram_partial -s 1 -c 1 python scripts/step_once.py --config S1 --steps 2 > gpurun_out/g6/ncu_S1.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gram_partial -s 1 -c 1 python scripts/step_once.py --config C3 --steps 2 > gpurun_out/g6/ncu_C3.txt 2>&1
for C in S1 C3 C4; do timeout 300 python bench.py --config $C --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/g6/bench_$C.json 2>&1; done
