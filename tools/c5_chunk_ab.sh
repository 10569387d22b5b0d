for r in 1 2; do for ch in ${CHUNKS:-32 64 128}; do
SWE_EARLY_CHUNK=$ch timeout 300 python bench.py --config c5 --steps 300 --warmup 5 --no-cpu-baseline --no-parity --e2e-steps 2 --fast 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$r chunk $ch', '%.4f ms'%d['ms_per_step'], d['activity']['active_fraction'], d['roofline']['frac'], d['clocks'].get('sm_mhz'))"
done; done
