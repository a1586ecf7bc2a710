RUN_PARITY=1 NO_FIELD=1 bash tools/exp_variant.sh ts "" "-DSE1P_MODES_TWO_STREAMS=0"
timeout 300 python tools/graph_times.py 2>&1 | tail -5
