# Tile-kernel experiments (SE1P_TILE_DBG bit 2: consumers skip the k-steps)
for d in 0 2; do echo "dbg=$d"; SE1P_TILE_DBG=$d timeout 300 python tools/stage_times.py ${1:-C5}; done
