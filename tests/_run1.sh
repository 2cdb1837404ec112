for ms in 6 8 10 12 16 24 32; do echo "min_steps $ms"; python - <<PY
import sys
sys.path.insert(0, ".")
import runpy
import paper_1612_00530_b200 as sp
sp.set_option("ring_min_steps", $ms)
sys.argv=["x"]
src=open("tests/hybrid_probe.py").read().split('timeit(pc, "hybrid, one kernel')[0]
exec(src)
PY
done
