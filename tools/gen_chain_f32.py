"""Regenerate csrc/chain_f32.cuh (float32 chain rule for the training step)
from the float64 sources: project_core (common.cuh) and chain_one
(project.cu), statement for statement with float32 types and literals,
expf for the glibc exp port, float copies of the camera and constants.

    python tools/gen_chain_f32.py
"""

import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2509_05216_b200", "csrc")


def conv(src: str) -> str:
    s = src.replace("double", "float")
    s = re.sub(r"(?<![\w.])(\d+\.\d*(?:e-?\d+)?)(?![\w.])", r"\1f", s)
    s = s.replace("exp_glibc(", "expf(")
    for c in ("NEAR_PLANE", "COV_DILATION", "SH_C0", "SH_C1"):
        s = s.replace(c, c + "_F")
    s = s.replace("const Cam &cam", "const CamF &cam")
    s = s.replace("Proj &o", "ProjF &o").replace("Proj o;", "ProjF o;")
    s = s.replace("bool project_core(", "bool project_core_f32(")
    s = s.replace("project_core<P>(", "project_core_f32<P>(")
    s = s.replace("bool chain_one(", "bool chain_one_f32(")
    s = s.replace("const Row<P> &in", "const RowF &in").replace("const Row<P> &row", "const RowF &row")
    s = s.replace("Grads &out", "GradsF &out").replace("zero_grads(out);", "zero_grads_f32(out);")
    s = s.replace("const float *g2", "const double *g2")
    return s


def main():
    common = open(os.path.join(CSRC, "common.cuh")).read()
    proj = open(os.path.join(CSRC, "project.cu")).read()
    head = open(os.path.join(CSRC, "chain_f32.cuh")).read()
    pc = common[common.index("template <typename P>\n__device__ __forceinline__ bool project_core("):
                common.index("inline int blocks_for(")]
    ch = proj[proj.index("template <typename P>\n__device__ __forceinline__ bool chain_one("):
              proj.index("// rasterizer.py:248-280 (chain_to_params)")]
    ps = common[common.index("struct Proj {"):common.index("template <typename P>\nstruct Row {")]
    prefix = head[:head.index("struct ProjF {")]
    out = prefix + conv(ps).replace("struct Proj {", "struct ProjF {") + conv(pc) + conv(ch)
    out += "\n}  // namespace isg\n"
    open(os.path.join(CSRC, "chain_f32.cuh"), "w").write(out)


if __name__ == "__main__":
    main()
