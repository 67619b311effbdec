"""Profile helper: C5 scene, one forward step (k=0), used under ncu."""
import sys
sys.path.insert(0, '.')
import bench
from paper_2603_16478_b200 import forward as fw, core
sc = bench.make_scene(int(sys.argv[1]), fingers=True)
sm = core.assemble_system_matrix(sc)
st = sc.rest_state()
for k in range(int(sys.argv[2])):
    bench.move_fingers(sc, k)
    st, rep = fw.forward_step(sc, st, sm, fw.ForwardConfig())
    print(k, rep.iterations, rep.krylov_iterations)
