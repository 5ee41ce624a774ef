set -x
timeout 300 python -m pytest tests/test_gpu_persistent.py -q -x -p no:cacheprovider -k bitwise 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_faces.py tests/test_gpu_report.py tests/test_gpu_persistent.py -q -x -p no:cacheprovider 2>&1 | tail -5
timeout 600 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2e_c1.json 2> gpurun_out/r2e_c1.err; echo bench=$?
python -c "
import json;d=json.loads(open('gpurun_out/r2e_c1.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['roofline']['achieved'], d['roofline']['frac'], d.get('parity'), d['kernels'])"
