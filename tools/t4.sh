for i in 1 2; do
timeout 600 python bench.py --config c3 --warmup 3 --skip-insitu --skip-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', d['value'], d['e2e']['value'])"
OPENBLAS_NUM_THREADS=1 timeout 600 python bench.py --config c3 --warmup 3 --skip-insitu --skip-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3 ob1', d['value'], d['e2e']['value'])"
done
