import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
import profiles_tools as pt
regions = [(1,245,"helpers"),(245,290,"setup"),(290,339,"frame-start"),(339,365,"select"),(365,379,"count/prune"),(379,387,"pl"),(387,466,"switch"),(466,491,"beta-climb"),(491,527,"complete/crc"),(527,537,"descent-setup"),(537,559,"alpha-smem"),(559,602,"alpha-reg"),(602,631,"node-setup"),(631,670,"sum-node"),(670,727,"r1/spc-node"),(727,740,"cand-dpm"),(740,773,"c1-write"),(773,819,"insert"),(819,850,"replace"),(850,881,"output")]
agg, tot, totS, per_line = pt.source_regions(sys.argv[1], "decode.cu", regions)
for k,v in sorted(agg.items(), key=lambda x:-x[1][0]):
    print(f"{k:20s} inst {v[0]/tot*100:5.1f}%  stall {v[1]/totS*100:5.1f}%")
src=open("/root/repo/paper_1809_03606_b200/csrc/decode.cu").read().split("\n")
print("top lines")
for k,v in sorted(per_line.items(), key=lambda x:-x[1][0])[:40]:
    print(k, f"{v[0]/tot*100:5.2f}% st {v[1]/totS*100:5.2f}%", src[k-1].strip()[:90])
