export HG_CACHE_DIR=/tmp/hgcache_r2c
set -x
HG_B0_TILE_STAGES=2 python -m pytest tests/test_gpu_b0split.py -m gpu -x -q 2>&1 | tail -3
for c in 5-16 4; do python tools/prof_stages.py $c 2>&1 | grep -v Warn; done
python - <<'P'
import paper_2406_06283_b200 as hg
from paper_2406_06283_b200 import cache
for c in ("4","5-16"):
    pre, P, info = cache.solver_for_config(c)
    print(c, "hit", info["hit"], pre._meta.get("tune"))
P
