"""Static check of the programmatic-dependent-launch contract in the built kernels: list the global memory
instructions each kernel issues before its griddepcontrol.wait (SASS ACQBULK). Only loads of data that no
kernel of the same decode chain writes may appear there (the index's centroid ids in scan, the caller's hot
rows in qprep and attend_partial, the query in the top-k kernel); a load of a predecessor's output hoisted
above the wait (e.g. through a const __restrict__ pointer, which lets the compiler use the non-coherent
path and move the load) is a race, and so is any global store or atomic there.

    python scripts/check_pdl_sass.py [build dir]  -> prints {kernel: [pre-wait LDG lines]}
"""
import json
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = sys.argv[1] if len(sys.argv) > 1 else os.path.join(HERE, "..", "paper_2602_07721_b200", "build")


def prewait_loads(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    res = {}
    for blk in re.split(r"\n\s*Function : ", out)[1:]:
        name = blk.split("\n", 1)[0].strip()
        if "ACQBULK" not in blk:
            continue
        pre = blk.split("ACQBULK", 1)[0]
        loads = [re.sub(r"\s+", " ", l.split("*/", 1)[1]).strip(" ;") for l in pre.split("\n")
                 if re.search(r"\b(LDG|STG|ATOMG|REDG|RED|ATOM)(\.|\s)", l) and "*/" in l]
        res[name] = loads
    return res


def main():
    allres = {}
    for f in ("qprep.cu.o", "scan.cu.o", "rerank.cu.o", "attend.cu.o", "postings.cu.o"):
        p = os.path.join(BUILD, f)
        if os.path.exists(p):
            allres.update(prewait_loads(p))
    print(json.dumps(allres, indent=1))


if __name__ == "__main__":
    main()
