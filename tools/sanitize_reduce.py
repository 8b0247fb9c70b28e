"""Small runs of the TMA neighbour reduce for compute-sanitizer (memcheck / racecheck /
synccheck): every relation with the default shape, a static alternative and the
dynamically dealt shapes (tsg_set_reduce_variant), each checked against the oracle.
    compute-sanitizer --tool racecheck python tools/sanitize_reduce.py [RxCxK]"""
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import tsg_oracle as O  # noqa: E402
import paper_1908_06094_b200 as T  # noqa: E402
from paper_1908_06094_b200 import _lib  # noqa: E402

r, c, k = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "21x40x35").split("x"))
spec = T.PatchSpec(r, c, k)
rng = np.random.default_rng(3)
n = 0
for (f, t) in T.OFFSET_TABLES:
    src = T.make_storage(spec, t, "a")
    dst = T.make_storage(spec, f, "b")
    a = rng.random((T.element_count(spec, t), k))
    T.flat_to_field(a, src)
    want = O.neighbor_sum(O.neighbor_table(r, c, f.value, t.value), a)
    for v in (0, 2, 11, 12, 16):
        _lib.call("tsg_set_reduce_variant", v)
        T.run_gpu(T.build_reduce(spec, f, t, src, dst))
        assert np.array_equal(T.field_to_flat(dst), want), (f, t, v)
        n += 1
_lib.call("tsg_set_reduce_variant", 0)
torch.cuda.synchronize()
print(f"sanitize_reduce: {n} launches bitwise == oracle")
