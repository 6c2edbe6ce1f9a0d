import faulthandler, sys, time, os
sys.argv = ["emu_worker.py"] + sys.argv[1:]
sys.path.insert(0, "tests")
faulthandler.dump_traceback_later(4, repeat=True, exit=False)
import emu_worker
t0 = time.time()
try:
    emu_worker.main()
finally:
    print("elapsed", time.time() - t0, file=sys.stderr)
