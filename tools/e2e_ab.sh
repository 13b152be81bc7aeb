for c in 0 4 0 4; do
  python bench.py --skip-extras --steps 10 --e2e-chunk $c --cpu-sample 1 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('chunk', $c, round(d['e2e']['value'],2), round(d['e2e']['pcie_floor'],2))"
done
