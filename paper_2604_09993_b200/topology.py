"""Compile-time model topology: the key that selects a kernel instantiation.

The CUDA kernels are templated on a model's *topology* (link/joint/contact
structure, surface kind, path-constraint structure, number of mixed path
channels) so that every index is a compile-time constant and the sparse
Jacobian patterns of the maximal-coordinate dynamics unroll into straight-line
fp64 code.  Numeric parameters (masses, anchors, gravity, mixing values, ...)
stay runtime kernel parameters, so e.g. all point-mass variants of the
reference tests share one instantiation.

``topology_key`` must produce the same string as ``topo_key()`` in
csrc/cito_capi.cu (computed from the packed ``cito_model_desc``).
"""

# Topologies compiled into the library (csrc/gen_models.py reads this list).
# Each entry: (name, n_links, joints[(parent, child, actuated)], contact_links,
#              implicit_surface, n_g_out, joint_limit_joints, height_bound_links)
_HC_JOINTS = ((0, 1, 1), (1, 2, 1), (2, 3, 1), (0, 4, 1), (4, 5, 1), (5, 6, 1))
_BIPED_JOINTS = ((0, 1, 1), (1, 2, 1), (0, 3, 1), (3, 4, 1))

COMPILED = [
    ("freelink", 1, (), (), False, 0, (), ()),
    ("pointmass", 1, (), (0,), False, 0, (), ()),
    ("pointmass_g1", 1, (), (0,), False, 1, (), ()),
    ("sinusoid", 1, (), (0,), True, 0, (), ()),
    ("sinusoid_g1", 1, (), (0,), True, 1, (), ()),
    ("pendulum", 1, ((-1, 0, 0),), (), False, 0, (), ()),
    ("dpendulum", 2, ((-1, 0, 0), (0, 1, 1)), (), False, 0, (), ()),
    ("monoped", 2, ((0, 1, 1),), (1,), False, 0, (), ()),
    ("monoped_g1", 2, ((0, 1, 1),), (1,), False, 1, (), ()),
    ("biped", 5, _BIPED_JOINTS, (2, 4), True, 0, (), ()),
    ("biped_g2", 5, _BIPED_JOINTS, (2, 4), True, 2, (), ()),
    ("halfcheetah", 7, _HC_JOINTS, (3, 6), False, 0, (), ()),
    ("halfcheetah_g2", 7, _HC_JOINTS, (3, 6), False, 2, (), ()),
]


def key_from_parts(n_links, joints, contact_links, implicit, n_g_out, jl_joints, hb_links):
    js = ",".join(f"{p}>{c}{'a' if a else 'p'}" for p, c, a in joints)
    cs = ",".join(str(c) for c in contact_links)
    jl = ",".join(str(j) for j in jl_joints)
    hb = ",".join(str(l) for l in hb_links)
    return f"L{n_links}|J{js}|C{cs}|S{'i' if implicit else 'f'}|G{n_g_out}|JL{jl}|HB{hb}"


def key_from_desc(desc):
    joints = [(desc.joint_parent[j], desc.joint_child[j], desc.joint_actuated[j]) for j in range(desc.n_joints)]
    contacts = [desc.contact_link[i] for i in range(desc.n_contacts)]
    jl = [desc.jl_joint[k] for k in range(desc.n_joint_limits)]
    hb = [desc.hb_link[k] for k in range(desc.n_height_bounds)]
    return key_from_parts(desc.n_links, joints, contacts, desc.surface_kind == 1, desc.n_g_out, jl, hb)


def compiled_keys():
    return {key_from_parts(*e[1:]): e[0] for e in COMPILED}


def entry_from_desc(desc, name=None):
    """A COMPILED-style entry for the topology of a packed model (any RobotModel
    within the kernel limits): what the JIT build (build.build_topology) compiles
    when the bundled library does not carry it."""
    import hashlib

    joints = tuple((int(desc.joint_parent[j]), int(desc.joint_child[j]), int(desc.joint_actuated[j]))
                   for j in range(desc.n_joints))
    contacts = tuple(int(desc.contact_link[i]) for i in range(desc.n_contacts))
    jl = tuple(int(desc.jl_joint[k]) for k in range(desc.n_joint_limits))
    hb = tuple(int(desc.hb_link[k]) for k in range(desc.n_height_bounds))
    key = key_from_desc(desc)
    if name is None:
        name = "jit_" + hashlib.sha1(key.encode()).hexdigest()[:12]
    return (name, int(desc.n_links), joints, contacts, desc.surface_kind == 1, int(desc.n_g_out), jl, hb), key
