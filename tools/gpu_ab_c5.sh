for i in 1 2; do
for lib in "" "GSS_LIB=build/libgss_old.so"; do
  echo "lib=${lib:-new}"; env $lib timeout 600 python tools/c5_emulate.py --rows-per-shard 2000000 --p 64 --shards 2 4 --cycles 4 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print([(r['shards'], r['sharded_us_per_coordinate'], r['unsharded_us_per_coordinate_same_total_rows']) for r in d['runs']])"
done; done
