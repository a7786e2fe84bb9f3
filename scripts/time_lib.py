"""kernel_times.py against another library build: python scripts/time_lib.py LIB B H N d alpha causal"""
import os, sys, runpy
os.environ["ENTMAX_ATTN_LIB"] = os.path.abspath(sys.argv[1])
sys.argv = [sys.argv[0]] + sys.argv[2:]
runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "kernel_times.py"), run_name="__main__")
