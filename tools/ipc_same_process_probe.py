"""Diagnostic: two stages in one process over gp_link_ipc (UVA path), progress per epoch."""
import faulthandler, os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2308_10087_b200 as gp
import ipc_stage_worker as W
faulthandler.dump_traceback_later(45, exit=True)
S = 2
ds, model, chunk_of = W.problem()
engs = [W.stage_engine(ds, model, chunk_of, r, S, 0) for r in range(S)]
blobs = [e.ipc_export() for e, _ in engs]
engs[0][0].link_ipc(None, blobs[1][0])
engs[1][0].link_ipc(blobs[0][1], None)
print("linked", flush=True)
mode = sys.argv[1] if len(sys.argv) > 1 else "threads"
def run(r, epochs):
    for t in range(1, epochs + 1):
        t0 = time.time()
        engs[r][0].run_epoch(t, gp.shuffle_chunk_order(W.K, t, 1))
        print(f"stage {r} epoch {t} done {time.time() - t0:.3f}s", flush=True)
th = [threading.Thread(target=run, args=(r, 3)) for r in range(S)]
for t in th: t.start()
for t in th: t.join()
print("all done", flush=True)
