"""Generate tests/golden/ref_prior_golden.noma (+ .summary.txt) with the
REFERENCE ITSELF: noma::save_prior (prior_bundle.cpp:103-139) and
noma::prior_summary (199-220) of the unmodified reference sources
(oracle/_ref/libnoma_ref.so) on the seeded bundle of tests/prior_cases.py.
tests/test_prior.py checks paper_2503_01582_b200.prior against these where the
compiled reference is absent. Re-run: python tests/golden/make_golden_prior.py
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle import pyoracle  # noqa: E402
from prior_cases import golden_bundle_inputs  # noqa: E402


def main():
    pyoracle.build_oracle(ref=True)
    ref = pyoracle.Ref()
    arch, theta, grid, verts, tris, prov = golden_bundle_inputs()
    out = Path(__file__).with_name("ref_prior_golden.noma")
    ref.save_prior(out, prov["category"], arch, theta, grid, verts, tris, search_seed=prov["search_seed"],
                   population=prov["population"], generations=prov["generations"],
                   genome_ints=prov["genome_ints"], genome_floats=prov["genome_floats"])
    st, text = ref.prior_summary(out)
    assert st == 0, text
    out.with_suffix(".summary.txt").write_text(text)
    print("wrote", out, out.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
