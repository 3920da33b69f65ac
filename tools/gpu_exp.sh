for k in 0 3 6; do
  echo "=== keep0=$k"
  CD_KEEP0=$k timeout 120 python tools/timeline.py dc 0.9 2>&1 | tail -4
done
