set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
cat > /tmp/rc.py <<'PY'
import sys, json
sys.path.insert(0, '.')
from paper_2407_11488_b200.cuda_backend import CudaTarget
from paper_2407_11488_b200.measure import MeasurementProtocol
from paper_2407_11488_b200.problems import make_problem
from paper_2407_11488_b200.paramspace import config_key
prob = make_problem("hotspot")
tgt = CudaTarget(prob, verify=False)
for c in sys.argv[1].split(";"):
    c = tuple(int(x) for x in c.split(","))
    o = tgt.execute(c, MeasurementProtocol(warmup_runs=1, benchmark_runs=7, flush_l2=True))
    print(json.dumps({"config": c, "time_ms": o.time_ms, "launch_ms": tgt.extras[config_key(c)].get("launch_ms")}))
PY
timeout 600 python /tmp/rc.py "$1" > gpurun_out/noverify.jsonl 2> gpurun_out/noverify.err
