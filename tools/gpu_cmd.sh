NO_FIELD=1 RUN_PARITY=1 bash tools/exp_variant.sh un "-DSE1P_GATHER_UNROLL=2"
