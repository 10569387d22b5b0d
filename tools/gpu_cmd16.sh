for r in 1 2 3; do for c in d8k c2; do
timeout 300 python bench.py --steps 1000 --warmup 20 --config $c --no-cpu-baseline --e2e-steps 2 --fast 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['clocks']; print('$r $c fast', '%.4f ms'%d['ms_per_step'], d['roofline']['frac'], k.get('sm_mhz'), k.get('reasons'))"
done; done
for c in d8k; do SWE_GUIDED=0 timeout 300 python bench.py --steps 1000 --warmup 20 --config $c --no-cpu-baseline --e2e-steps 2 --fast 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c unguided', '%.4f ms'%d['ms_per_step'])"; done
