RUN_PARITY=1 bash tools/exp_variant.sh fp "" "-DSE1P_FIELD_ONE_PASS=1"
