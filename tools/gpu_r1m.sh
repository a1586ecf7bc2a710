set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1m_pytest.log 2>&1
tail -3 gpurun_out/r1m_pytest.log
bash tools/tile_experiments.sh C5 > gpurun_out/r1m_exp.log 2>&1
cat gpurun_out/r1m_exp.log
