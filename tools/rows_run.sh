set -x
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/rows_smoke.log 2>&1; tail -2 gpurun_out/rows_smoke.log
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/rows_pytest.log 2>&1; tail -3 gpurun_out/rows_pytest.log
for zc in 0 8 16 32; do
  if [ $zc = 0 ]; then E=""; else E="RKB_ZCHUNK=$zc"; fi
  env $E timeout 600 python bench.py --legs euler,midpoint,rk4,ab1,ab2,ab4,adaptive --steps 5 > gpurun_out/rows_zc$zc.log 2>&1
  grep -oE '"(leg|metric)": "[^"]*"|"frac": [0-9.]+' gpurun_out/rows_zc$zc.log | head -40
done
