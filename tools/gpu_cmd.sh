bash tools/exp_variant.sh il "-DSE1P_DMMA_INTERLEAVE=1" "-DSE1P_DMMA_INTERLEAVE=0"
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_field.py -x -q 2>&1 | tail -3
