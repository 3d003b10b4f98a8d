"""A small multi-element-per-CTA case for compute-sanitizer (racecheck / synccheck / memcheck), one tool per call:

    HDG_MAX_GRID=4 compute-sanitizer --tool racecheck python tools/sanitize_case.py C4

The persistent grid is capped (HDG_MAX_GRID) so every CTA condenses several elements: the TMA / mbarrier /
named-barrier pipeline of the element loop runs, half of the elements fail the speculative GEPP check (rows
permuted: the exact path runs while the next element's loads are in flight) and one is singular. The results are
checked against the oracle, so a run that the tool lets finish must also be correct."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import gen
    import oracle
    from gpu_helpers import run_gpu
    from test_pivot_fullpath_gpu import check_perturbed
    cases = {"C4": dict(m_elem=12, p_fixed=3, nr=2, nt=8), "C3": dict(m_elem=4, p_fixed=4, nr=2, nt=8),
             "C2": dict(m_elem=4, p_fixed=2, nr=4, nt=16), "NSp4": dict(m_elem=12, p_fixed=4, nr=2, nt=4)}
    names = sys.argv[1:] or ["C4"]
    for name in names:
        c = cases[name]
        w = gen.make_workload(name, nr=c["nr"], nt=c["nt"], m_elem=c["m_elem"], p_fixed=c["p_fixed"],
                              seed=gen.SEED_BASE + 9)
        worst = check_perturbed(w, seed=77)
        print(f"sanitize case {name}: E={w.E} grid cap={os.environ.get('HDG_MAX_GRID')} ok {worst}", flush=True)
    _ = (oracle, run_gpu, np)


if __name__ == "__main__":
    main()
