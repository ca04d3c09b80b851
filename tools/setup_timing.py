"""Host setup cost (generator, factor, device pack) of the bench trees."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_01745_b200 as so
print("nproc", os.cpu_count(), flush=True)
for br in ([8, 8, 8, 2], [16, 8, 8, 2], [64, 8, 8, 2], [8, 8, 8, 8, 4]):
    t0 = time.time(); p = so.gen_random_instance(1, 50, 20, 20, br); t1 = time.time()
    c = so.factor(p); t2 = time.time()
    c.device(); t3 = time.time()
    print(br, p.num_nodes(), f"gen {t1-t0:.1f}s factor {t2-t1:.1f}s dev {t3-t2:.1f}s", flush=True)
    del c, p
