for r in 1 2 3; do
  for v in base k3gen; do
    echo "$v $(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/prefill_breakdown.py --reps 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['k3_vs_ms'],2))")"
  done
done
