for cfg in "A=1 L=1 R=1" "A=1 L=4 R=4" "A=1 L=2 R=2" "A=1 L=4 R=2"; do
  echo "== $cfg"; timeout 120 python tools/e2e_timeline.py $cfg 2>&1 | tail -2
done
