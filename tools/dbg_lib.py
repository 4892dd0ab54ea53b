"""Run a script against an alternative in-tree build of the library: dbg_lib.py LIB script.py [args]"""
import runpy, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_04569_b200 import _native as N
N.LIB_PATH = os.path.abspath(sys.argv[1])
N.load.__defaults__ = (N.LIB_PATH,)
sys.argv = sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
