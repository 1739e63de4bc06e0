import cProfile, pstats, sys, io
sys.argv=['x']
sys.path.insert(0,'tools'); sys.path.insert(0,'.')
import c1_breakdown
pr=cProfile.Profile(); pr.enable(); c1_breakdown.main(); pr.disable()
s=io.StringIO(); pstats.Stats(pr,stream=s).sort_stats('tottime').print_stats(25); print(s.getvalue()[:6000])
