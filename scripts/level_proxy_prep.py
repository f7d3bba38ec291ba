"""Level table + tip codes of the dengue workload for scripts/level_proxy.cu
(post levels by height, pre levels by depth; entries (node, child a, child b))."""
import os, struct, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import phylo_synth as ps  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/level_proxy_dengue.bin"
pb = ps.config1_dengue()
N, C, R, ops = pb.n_tips, pb.patterns, len(pb.cat_rates), np.asarray(pb.ops)
height, depth = {}, {ops[-1][0]: 0}
for d, a, b in ops:
    height[d] = 1 + max(height.get(a, 0), height.get(b, 0))
for d, a, b in ops[::-1]:
    depth[a] = depth[b] = depth[d] + 1
post, pre = {}, {}
for d, a, b in ops:
    post.setdefault(height[d], []).append((d, a, b))
    pre.setdefault(depth[d], []).append((d, a, b))
with open(out, "wb") as f:
    f.write(struct.pack("5i", N, C, R, len(post), len(pre)))
    for lv in (post, pre):
        for key in sorted(lv):
            e = np.asarray(lv[key], dtype=np.int32)
            f.write(struct.pack("i", len(e)))
            f.write(e.tobytes())
    f.write(np.asarray(pb.tip_states, dtype=np.int8).tobytes())
print(out, len(post), len(pre))
