export HG_CACHE_DIR=/tmp/hgcache_r2d
set -x
python tools/prof_stages.py 5-32 2>&1 | grep -v Warn
python - <<'P'
import paper_2406_06283_b200 as hg
from paper_2406_06283_b200 import cache
for c in ("5-32",):
    pre, P, info = cache.solver_for_config(c)
    print(c, "hit", info["hit"], pre._meta.get("tune"), pre._meta.get("b0_split_dev"), pre._meta.get("b0_split_extended"), pre._meta.get("b0s_ns"))
    print(P.times)
P
python -m pytest tests/test_gpu_b0split.py tests/test_gpu_large.py -m gpu -x -q -k "b0split or 5-32" 2>&1 | tail -3
