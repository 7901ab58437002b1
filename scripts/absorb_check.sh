# absorbed-path (f4 (ii)) parity tests + cfg4 bench line + per-kernel ncu list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k absorbed --timeout 300 2>&1 | tail -3
timeout 300 python bench.py --absorb --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/absorb_cfg4.json 2>gpurun_out/absorb_cfg4.err; tail -3 gpurun_out/absorb_cfg4.err
python -c "
import json;d=json.loads(open('gpurun_out/absorb_cfg4.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['value'],d['kernels']['absorbed_hidden'],d['roofline']['frac'],d['clocks'])"
bash scripts/absorb_ncu.sh
