# Tile-kernel experiments (SE1P_TILE_DBG bits: 1 no DMMA, 2 no k-steps, 4 no list building)
for d in 0 1 2 6; do echo "dbg=$d"; SE1P_TILE_DBG=$d timeout 300 python tools/stage_times.py ${1:-C5}; done
