# A/B of the table build: default lib vs a variant (argument), cfg2 and cfg5,
# serial tables (TNB_TABLE_STREAM=0) so the table time is its own
for i in 1 2; do
for L in "" "$1"; do
 for E in "TNB_TABLE_STREAM=1" "TNB_TABLE_STREAM=0"; do
 echo "== lib=$L $E"; env TNB_LIB=$L $E timeout 200 python bench.py --steps 10 --warmup 3 --no-secondary --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['other_kernels_ms'])"
 done
done; done
