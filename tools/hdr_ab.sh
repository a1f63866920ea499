# C3 header step (72 rows) with K5 v2 vs K4 (page-centric items) for its attention
for cfg in "CHOREO_WIDE_K4=0" "CHOREO_WIDE_K4=1"; do
  echo "== $cfg"; env $cfg timeout -s KILL 200 python tools/header_timing.py 2>&1 | tail -2
done
