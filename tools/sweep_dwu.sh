# Development: wide-FCN step time vs the SM budget of the overlapped dW + update (ST_DWU_SMS)
for S in 60 72 84 96 148; do
  echo "ST_DWU_SMS=$S $(ST_DWU_SMS=$S timeout 300 python bench.py --no-cpu --no-e2e --steps 60 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],3))')"
done
