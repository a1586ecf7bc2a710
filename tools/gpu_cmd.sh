NO_FIELD=1 RUN_PARITY=1 bash tools/exp_variant.sh nb "" "-DSE1P_GRID_NOBRANCH=1" "-DSE1P_GATHER_ACC2=1"
