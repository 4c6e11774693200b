import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = ["x", "c3a_or50", "4096", "1"]
import runpy
runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "exit_probe.py"), run_name="__main__")
time.sleep(3)
print("slept", flush=True)
