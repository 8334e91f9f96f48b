"""A paper-size Groth16 key setup (comb-based base generation): for ncu."""
import sys

sys.path.insert(0, ".")
from paper_2603_10242_b200 import _native as N, groth16  # noqa: E402

pk = groth16.ProvingKey(groth16.PAPER_T, groth16.PAPER_K, ctx=N.context(0))
pk.close()
print("ok")
