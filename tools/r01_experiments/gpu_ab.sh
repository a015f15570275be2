for v in "1 1" "0 1" "1 0" "0 0"; do set -- $v; echo "full $1 prio $2"; export FKD_FULL_STAGING=$1 FKD_TAIL_PRIO=$2
python tools/e2e_diag.py 2>&1 | grep auto
python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value']/1e6, d['e2e']['value']/1e6)"
done
