"""Build libsft variants (-D overrides of the translation kernel configs) into sweep_libs/."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0801_1524_b200 import build as b  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VARIANTS = {
    # name: list of -D flags
}


def parse(spec):
    """'G29=8,NC29=8,MINB29=2' -> ['-DSFT_WS_G29=8', ...]; keys starting with NSUB map to SFT_NSUB*"""
    out = []
    for kv in spec.split(","):
        k, v = kv.split("=")
        out.append(f"-DSFT_{k}={v}" if k.startswith(("NSUB", "TAIL", "ROTATE", "ABSENT", "CENTRE", "ABL_", "TMA_", "PAD_", "LEAF_", "FINAL_", "SLOTPAD", "CLASS_", "F32", "PRODUCER", "INSTR", "BS_", "SORT_", "TREE_", "CLUSTER_", "F2_", "ORDER3", "ROUND_", "PL", "SYM5", "TAIL5", "PUBLISH", "CNT3", "CLASS_SPLIT3")) else f"-DSFT_WS_{k}={v}")
    return out


if __name__ == "__main__":
    os.makedirs(os.path.join(ROOT, "sweep_libs"), exist_ok=True)
    specs = sys.argv[1:]
    def one(spec):
        name = "lib_" + spec.replace(",", "_").replace("=", "") + ".so"
        b.build(extra=parse(spec), out=os.path.join(ROOT, "sweep_libs", name))
        return name
    with ThreadPoolExecutor(4) as ex:
        for n in ex.map(one, specs):
            print(n)
    # the variants' objects are not needed once linked (keep the gpurun snapshot small)
    import glob
    for o in glob.glob(os.path.join(ROOT, "paper_0801_1524_b200", "build", "*_*.o")):
        os.remove(o)
