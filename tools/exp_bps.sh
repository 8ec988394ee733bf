for b in 1 2 4; do for c in c4 c5; do GP_TOPR_BPS=$b timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); print('bps $b', '$c', d['ms_per_step'])"; done; done
