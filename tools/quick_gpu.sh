# smoke + GPU parity + bench legs; usage: tools/quick_gpu.sh TAG "legs" [extra env]
TAG=$1; LEGS=${2:-euler,midpoint,rk4,ab1,ab2,ab4,adaptive}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; tail -1 gpurun_out/${TAG}_pytest.log
env $3 timeout 600 python bench.py --legs $LEGS --steps 5 > gpurun_out/${TAG}_bench.log 2>&1
python tools/legs_table.py gpurun_out/${TAG}_bench.log
