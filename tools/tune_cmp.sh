timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
bash tools/tune.sh "" def; python tools/tune_table.py gpurun_out/tune_def.csv | head -7
bash tools/zc_sweep.sh zs euler,midpoint,rk4,ab1,ab2,ab4,adaptive "6,16,32,48 8,16,32,48 12,16,32,48 16,16,32,48"
