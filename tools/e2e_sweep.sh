# e2e (host buffers, copies in the timed region) vs the number of e2e steps and applies in flight
for args in "--e2e-steps 100" "--e2e-steps 400" "--e2e-steps 400 --streams 16"; do
  timeout 400 python bench.py --steps 400 --warmup 3 --no-cpu-baseline --gmres-maxit 0 $args 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$args', 'K=%d value %.0f e2e %.0f GB/s (%.4f ms/step)' % (d['config']['concurrency'], d['value'], d['e2e']['value'], d['e2e']['ms_per_step']), flush=True)"
done
