import json,sys
d=json.load(open(sys.argv[1]))
print(round(d["value"]),round(d["ms_per_step"],1),round(d["roofline"]["frac"],3),round(d["fused_roofline"]["frac"],3), d["clocks"]["sm_mhz"])
print({k:(v["launches"],round(v["ms_per_step"],1),round(v.get("tflops",0),1)) for k,v in d["kernels"].items()})
