"""Times arbitrary (dims, blocks) shapes on 1 GPU: python tools/perf_shapes.py 512x512x512:16x16x16 ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_12734_b200 as jb
iters = int(os.environ.get("ITERS", 40))
flags = int(os.environ.get("FLAGS", 0))
for spec in sys.argv[1:]:
    d, b = spec.split(":")
    dims = tuple(int(v) for v in d.split("x")); blocks = tuple(int(v) for v in b.split("x"))
    with jb.Jacobi3D(dims, blocks, flags=flags) as s:
        s.set_init_hash(1)
        s.step(4)
        s.step(iters)
        ms = s.last_step_ms() / iters
        sw = s.profile_sweep(5)
        pts = dims[0] * dims[1] * dims[2]
        st = s.stats()
        print(f"{spec:28s} ext={s.block_extent} {ms*1e3:9.1f} us/iter {pts/(ms*1e6):7.1f} GLUP/s "
              f"{16*pts/(ms*1e6):6.0f} GB/s sweep {sw*1e3:8.1f} us variant={st['sweep_variant']} blocks={st['local_blocks']}", flush=True)
