"""Executed warp instructions / stall samples of k_raycast grouped by code
region (regions located by marker strings in raycast.cu, so the grouping
survives edits).  usage: python tools/ncu_buckets.py report.ncu-rep"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_lines import load  # noqa: E402

SRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2309_04393_b200", "csrc", "raycast.cu")
# (name, start marker, end marker): lines [start, end)
REGIONS = [
    ("tf_eval", "__device__ __forceinline__ void tf_eval(", "// kernels.py:97-116"),
    ("box_exit / axis_box", "// kernels.py:97-116", "// first-seen request:"),
    ("level_pos", "__device__ __forceinline__ void level_pos(", "#ifndef RO_META_HINT"),
    ("substitute", "__device__ __forceinline__ int2 substitute(", "// trilinear tap addresses"),
    ("taps_of", "__device__ __forceinline__ void taps_of(", "__device__ __forceinline__ double trilerp"),
    ("trilerp", "__device__ __forceinline__ double trilerp", "#ifndef RO_TAP_HINT"),
    ("load_taps", "__device__ __forceinline__ void load_taps", "// audit value"),
    ("lod_raw", "__device__ __forceinline__ int lod_raw(", "__device__ __forceinline__ int clampi("),
    ("pow_pow2", "__device__ __forceinline__ double pow_pow2(", "// raw LOD level"),
    ("classify kernels", "// Per-frame node classes for the residency walk", "__host__ __device__ constexpr int ilog2c"),
    ("staging", "    // ---- stage frame tables ----", "#if RO_PERSISTENT\n    // Persistent CTAs"),
    ("tile / packet setup", "#if RO_PERSISTENT\n    // Persistent CTAs", "    // Warp-uniform sample loop"),
    ("sample head (pos, LOD)", "    // Warp-uniform sample loop", "            // usage mask / histogram / per-pixel brick switches"),
    ("account", "            // usage mask / histogram / per-pixel brick switches", "            // Sub-block skip:"),
    ("sub_skip", "            // Sub-block skip:", "            auto finish = "),
    ("finish (taps, TF, composite ch)", "            auto finish = ", "            // taps + TF of the desired level"),
    ("sample lambdas", "            // taps + TF of the desired level", "            if (MODE == RO_MODE_PAGETABLE)"),
    ("baseline modes", "            if (MODE == RO_MODE_PAGETABLE)", "                // kernels.py:431-558 -- one cursor shared"),
    ("residency: leaf class", "                // kernels.py:431-558 -- one cursor shared", "#if RO_FAST_DESCENT"),
    ("residency: slow descent", "#if RO_FAST_DESCENT", "                // Fast path, channels 0..3"),
    ("residency: prefetch", "                // Fast path, channels 0..3", "                // one channel of the sample, in the reference's channel order"),
    ("residency: channel loop head + walk", "                // one channel of the sample, in the reference's channel order", "                    // at traversal depth: probe the desired brick"),
    ("residency: probe + request", "                    // at traversal depth: probe the desired brick", "                        // nearest resident level in this node"),
    ("residency: substitute call", "                        // nearest resident level in this node", "            if (skippable) {"),
    ("skip loop", "            if (skippable) {", "            } else {\n                stall = 0;"),
    ("composite", "            } else {\n                stall = 0;", "    // close every channel's last brick run"),
    ("pixel end + reductions", "    // close every channel's last brick run", "template <int MODE, bool CHECK, int BX, int BY, int BZ>\ncudaError_t launch_b"),
]


def line_of(src, marker):
    i = src.index(marker)
    return src.count("\n", 0, i) + 1


def main():
    per_line, _ = load(sys.argv[1])
    src = open(SRC).read()
    tot_i = sum(v[1] for v in per_line.values()) or 1
    tot_s = sum(v[0] for v in per_line.values()) or 1
    seen = set()
    print(f"{'region':40s} {'inst%':>6s} {'stall%':>7s}")
    for name, a, b in REGIONS:
        lo, hi = line_of(src, a), line_of(src, b)
        keys = [k for k in per_line if k[0] == "raycast.cu" and lo <= k[1] < hi]
        seen.update(keys)
        ins = sum(per_line[k][1] for k in keys)
        st = sum(per_line[k][0] for k in keys)
        print(f"{name:40s} {100 * ins / tot_i:6.1f} {100 * st / tot_s:7.1f}")
    rest = [k for k in per_line if k not in seen]
    ins = sum(per_line[k][1] for k in rest)
    st = sum(per_line[k][0] for k in rest)
    print(f"{'other (headers, unmatched lines)':40s} {100 * ins / tot_i:6.1f} {100 * st / tot_s:7.1f}")


if __name__ == "__main__":
    main()
