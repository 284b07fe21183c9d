# GPU validation pass: tests, smoke, short benches per config; outputs in gpurun_out/
export PYTHONPATH=$PWD
python -m pytest tests -x -q -m gpu > gpurun_out/t_check.log 2>&1; tail -3 gpurun_out/t_check.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_check.log 2>&1; tail -1 gpurun_out/smoke_check.log
python bench.py --config 2 --steps 5 --warmup 3 --no-cpu --no-probe > gpurun_out/s_c2.json 2> gpurun_out/s_c2.err
python bench.py --config 1 --steps 5 --warmup 3 --no-cpu --no-probe > gpurun_out/s_c1.json 2> gpurun_out/s_c1.err
python bench.py --config 3 --steps 3 --warmup 3 --no-cpu --no-probe > gpurun_out/s_c3.json 2> gpurun_out/s_c3.err
for m in ${MINBS:-6}; do
BVC_WALK3_MINB=$m python bench.py --config 4 --steps 2 --warmup 3 --no-cpu --no-probe > gpurun_out/m${m}_c4.json 2> gpurun_out/m${m}_c4.err
BVC_WALK3_MINB=$m python bench.py --config 5 --steps 2 --warmup 3 --no-cpu --no-probe > gpurun_out/m${m}_c5.json 2> gpurun_out/m${m}_c5.err
done
for f in s_c1 s_c2 s_c3 $(for m in ${MINBS:-6}; do echo m${m}_c4 m${m}_c5; done); do python -c "
import json;d=json.load(open('gpurun_out/$f.json'));print('$f',round(d['ms_per_step'],3),d['phases_s'],d['clocks']['sm_mhz'],d['clocks']['reasons'])"; done
