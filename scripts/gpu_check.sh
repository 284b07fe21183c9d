# GPU validation pass: tests, smoke, short benches per config; outputs in gpurun_out/
export PYTHONPATH=$PWD
python -m pytest tests -x -q -m gpu > gpurun_out/t_check.log 2>&1; tail -3 gpurun_out/t_check.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_check.log 2>&1; tail -1 gpurun_out/smoke_check.log
for c in 1 2 3 4 5; do
  python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-probe --no-extra > gpurun_out/s_c$c.json 2> gpurun_out/s_c$c.err
  python -c "
import json;d=json.load(open('gpurun_out/s_c$c.json'));print('c$c',round(d['ms_per_step'],3),d['phases_s'],d['clocks']['sm_mhz'],d['clocks']['reasons'])"
done
