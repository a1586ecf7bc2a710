for v in "" "SE1P_GATHER_BM=60 SE1P_GATHER_NB=5" "SE1P_GATHER_BM=56 SE1P_GATHER_NB=5"; do
  echo "== [$v]"; env $v timeout 200 python tools/stage_times.py C5 tiles; env $v timeout 200 python tools/stage_times.py C5 field; env $v timeout 200 python tools/stage_times.py C4 tiles
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
