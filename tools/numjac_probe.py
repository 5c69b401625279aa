"""C4 numeric-Jacobian timing alone (bench.py run_numjac), for A/B builds."""
import json
import sys
sys.path.insert(0, ".")
import bench
print(json.dumps(bench.run_numjac("c4")))
