timeout 600 python bench.py --config 32k --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/b32.json 2> gpurun_out/b32.err; echo rc $?
python -c "import json;d=json.load(open('gpurun_out/b32.json'));print(d['gpu_launches'], d.get('decode_tok_s_per_gpu'))"
tail -3 gpurun_out/b32.err
python - <<'PY'
import torch
from cuda.bindings import runtime as rt
print(rt.cudaGraphNodeType.cudaGraphNodeTypeKernel)
PY
