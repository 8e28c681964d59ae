import os, sys, subprocess
for flags in [0,1,2,4,8,16]:
    env=dict(os.environ, FF_DEBUG_FLAGS=str(flags))
    print("FLAGS", flags, flush=True)
    subprocess.run([sys.executable, "-c", """
import sys; sys.path.insert(0,'tests'); sys.argv=['x']
exec(open('tests/_probe_debug.py').read().split('for steps in')[0])
run(128, 4*128*2, 256, 1024, (4,1,128,256))
run(128, 8*128*3, 128, 2048, (8,1,128,256))
run(128, 4*64*3, 256, 1024, (4,1,64,256), gated=True)
"""], env=env, timeout=60)
