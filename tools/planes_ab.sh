make -C paper_2605_13928_b200/csrc -j16 > /dev/null 2>&1
for n in base f16 f16x1 bf16x1; do
  if [ $n = base ]; then L=; else L=$PWD/paper_2605_13928_b200/libscb_b200_$n.so; fi
  echo "== $n"
  SCB_LIB_PATH=$L timeout 900 python -m pytest tests/test_gpu_parity_scale.py -q -s -x -k "c2_parity_and or c3_parity_full" 2>&1 | grep -E "^parity|passed|failed|Error|assert" | head -6
  SCB_LIB_PATH=$L timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('bench', d['ms_per_step'], {k:v['ms'] for k,v in d['stages'].items()})"
done
