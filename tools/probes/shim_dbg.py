"""Debug run of one shim multi-rank case with FAKE_NCCL_DEBUG tracing (tests/test_gpu_shim_multirank.py)."""
import os
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)


def main():
    os.environ["FAKE_NCCL_DEBUG"] = "1"
    import test_gpu_shim_multirank as t
    import paper_2408_15384_b200 as mm
    cases = [(mm.MM_SUMMA_2D, "f64", 331, 389, 313, 0, 0, g, None) for g in ((1, 2), (2, 1))]
    cases.append((mm.MM_SUMMA_25D, "f64", 297, 450, 283, mm.MM_REPLICATE, 0, (1, 1), None))
    out = t._run(2, cases)
    t._check(2, cases, out)
    print("OK")


if __name__ == "__main__":
    main()
