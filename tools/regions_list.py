import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
import profiles_tools as pt
regions = [(1,100,"helpers"),(100,137,"setup/frame"),(137,171,"beta-climb"),(171,186,"alpha-smem"),(186,223,"alpha-reg"),(223,327,"node"),(327,365,"cand+c1"),(365,384,"publish"),(384,398,"prune"),(398,442,"transfer"),(442,500,"final")]
agg, tot, totS, per_line = pt.source_regions(sys.argv[1], sys.argv[2], regions)
for k,v in sorted(agg.items(), key=lambda x:-x[1][0]):
    print(f"{k:28s} inst {v[0]/tot*100:5.1f}%  stall {v[1]/totS*100:5.1f}%")
src=open("/root/repo/paper_1809_03606_b200/csrc/"+sys.argv[2]).read().split("\n")
print("top lines")
for k,v in sorted(per_line.items(), key=lambda x:-x[1][1])[:25]:
    print(k, f"{v[0]/tot*100:5.2f}% st {v[1]/totS*100:5.2f}%", src[k-1].strip()[:90])
