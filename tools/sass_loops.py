"""Static check of K1's loop bodies in a cubin / .so (cuobjdump): the loops that
contain the pass's 256-bit theta load, their length and how many special-register
reads / constant loads / moves the compiler put inside (register-pressure
rematerialisation shows up here first).  Usage: python tools/sass_loops.py lib.so"""
import re,subprocess,sys
# the full-corpus K1 variant (K <= 2048: 4 warps, 768-vector staging, 8
# CTAs/SM); its entry-parallel pass loop should stay ~104 SASS per step
DEFAULT_FN = "_ZN2gf13sample_kernelILi128ELj768ELi8ELb1ELb0EEEvNS_10SampleArgsE"


def loops(obj, fn=DEFAULT_FN):
    sass=subprocess.run(f"cuobjdump -sass {obj}",shell=True,capture_output=True,text=True).stdout
    i=sass.find("Function : "+fn); f=sass[i:sass.find("Function :",i+10)]
    ins=[]
    for l in f.split('\n'):
        m=re.match(r'\s+/\*([0-9a-f]{4})\*/\s+(.*?);',l)
        if m: ins.append((int(m.group(1),16), m.group(2).strip()))
    addr={a:k for k,(a,_) in enumerate(ins)}
    enl=[k for k,(a,s) in enumerate(ins) if 'ENL2.256' in s]
    for k,(a,s) in enumerate(ins):
        m=re.search(r'BRA(?:\.U)? (?:!?U?P\d+, )?(0x[0-9a-f]+)',s)
        if m:
            t=int(m.group(1),16)
            if t<a and t in addr and addr[t] <= enl[-1] <= k:
                body=ins[addr[t]:k+1]
                print(f"  loop {hex(t)}-{hex(a)} len={len(body)} S2R={sum('S2R' in x or 'S2UR' in x for _,x in body)} LDC={sum(x.startswith('LDC') or ' LDC' in x for _,x in body)} MOV={sum('MOV' in x for _,x in body)}")
for o in sys.argv[1:]:
    print(o); loops(o)
