import numpy as np, paper_1512_06126_b200 as emie
for (n, nz, hx) in [(12, 8, 100.0), (32, 32, 200.0)]:
    model = emie.LayeredModel([0.0, 800.0, 3000.0], [0.0, 0.05, 0.01, 0.2])
    breaks = list(np.linspace(900.0, 900.0 + 40.0 * nz, nz + 1))
    grid = emie.make_grid(model, breaks, n, n, hx, hx)
    sop = emie.assemble_operator(grid, model, 2 * np.pi * 3.0, keep_blocks=True)
    b = sop.blocks()
    ntri, nfull = nz*(nz+1)//2, nz*nz
    d = np.array([b[i, i] for i in range(n)])
    xx, yy = d[:, :ntri], d[:, ntri:2*ntri]
    xz, yz = d[:, 4*ntri:4*ntri+nfull], d[:, 4*ntri+nfull:]
    print(n, nz, "diag xx-yy", np.max(np.abs(xx-yy))/np.max(np.abs(xx)), "exact frac", np.mean(xx==yy),
          "xz-yz", np.max(np.abs(xz-yz))/np.max(np.abs(xz)), np.mean(xz==yz))
    per = [np.max(np.abs(xx[i]-yy[i]))/np.max(np.abs(b[i,i])) for i in range(n)]
    print("  per offset", ["%.1e" % p for p in per])
    # off-diagonal: mirror exactness
    off = max(np.max(np.abs(b[j, i] - np.concatenate([b[i,j,ntri:2*ntri], b[i,j,:ntri], b[i,j,2*ntri:4*ntri], b[i,j,4*ntri+nfull:], b[i,j,4*ntri:4*ntri+nfull]]))) for i in range(n) for j in range(i+1, n))
    print("  offdiag mirror max", off)
