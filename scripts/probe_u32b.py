import paper_2203_03732_b200 as otprg
inst = otprg.gen_uniform_square(64, 1)
try:
    m, s = otprg.solve_assignment(inst, otprg.AssignmentOptions(eps=0.05, storage="u32"))
    print("phases", s.phases)
except Exception as e:
    print(repr(e))
