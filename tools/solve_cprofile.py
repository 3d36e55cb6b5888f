"""cProfile of a config-3 BSFW solve (host-side hot spots)."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import run_solve  # noqa: E402

run_solve.run(3, "bsfw")  # warm (table build, allocations)
pr = cProfile.Profile()
pr.enable()
r = run_solve.run(3, "bsfw")
pr.disable()
print(r["solve_s"])
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
