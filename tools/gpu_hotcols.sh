for v in "" "--hot-cols" "--hot-cols --sort-rows" ""; do
  echo "== $v: $(timeout 300 python tools/profile_loop.py --config 2 --warmup 3 --periods 20 $v 2>&1 | grep -E 'periods:|Error|error' | head -3)"
done
