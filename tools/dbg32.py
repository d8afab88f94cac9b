import sys; sys.path[:0]=["tests","tests/golden","."]
import numpy as np
from parity_util import Case, sample_thetas
from paper_2310_07002_b200 import pcv
case=Case("logistic_loo")
c=pcv.Context(0); c.set_kernel_policy(c.KERNEL_TF32)
slot=c.add_model(case.models[0], case.kparams[0], case.banks[0], model_id=0)
th=sample_thetas(case,0,2,seed=0)
lp,g=c.eval(slot,[0,0],th)
og=case.omodels[0].grad(th[0],0)
np.set_printoptions(precision=4, linewidth=200, suppress=True)
print("dev ", g[0]); print("orc ", og); print("diff", g[0]-og); print("ratio", g[0]/og)
# also prior-free: G = grad + theta
print("G dev", g[0]+th[0]); print("G orc", og+th[0])
