import os
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libdacsr_b200.so")
