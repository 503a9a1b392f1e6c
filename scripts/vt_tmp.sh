mkdir -p gpurun_out/k1
timeout 900 python -m pytest tests -m gpu -q -x -k "graph or host or trajectory or sharding or set_grads or full_size" > gpurun_out/k1/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/k1/pytest.log
bash scripts/variant_phases.sh k1 "C1 C4 C2 C5 S1" nofork > gpurun_out/k1/phases.txt 2>&1
